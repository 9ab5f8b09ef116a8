"""A/B of Engine(xstream_pdl=...) on the BASELINE configs (GPU box): replay time,
parity against the fp32 CPU forward, bit-identity of the outputs.  profiles/r04_ab_xstream_pdl.txt"""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_02732_b200.engine as E
from paper_2012_02732_b200.networks import build_model, example_input
from oracle.numerics import cpu_forward
for cfg, bs in [('nasnet_mobile', 1), ('cell', 1), ('resnet50', 1), ('inception_v3', 1), ('nasnet_mobile', 256)]:
    model, shape = build_model(cfg)
    x = example_input(shape, batch=bs)
    ref = cpu_forward(model, x[:8])
    cache = f'/tmp/tune_{cfg}_{bs}.json'
    outs = {}
    for rnd in range(2):
        for xp in (False, True):
            eng = E.Engine(model, xstream_pdl=xp, tuning_cache=cache).prepare(x)
            eng.load_input_device(x)
            ts = [eng.time_replay(True, 200 if bs == 1 else 20)[0] for _ in range(3)]
            eng.replay(multi=True); eng.synchronize()
            y = eng.device_output().cpu().clone()
            ok = torch.allclose(y[:8].reshape(ref.shape), ref, rtol=1e-3, atol=1e-4)
            same = None if xp is False else torch.equal(y, outs[False])
            outs[xp] = y
            print(f"{cfg} bs{bs} xstream_pdl={xp}: replay us {' '.join(f'{t:.1f}' for t in ts)} parity {ok} bit-identical-to-off {same}", flush=True)
            eng.close()
