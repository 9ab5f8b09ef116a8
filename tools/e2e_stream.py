import sys, time, torch
sys.path.insert(0, '.')
from paper_2012_02732_b200.engine import Engine
from paper_2012_02732_b200.networks import build_model, example_input
m, s = build_model('nasnet_mobile')
xs = [example_input(s, seed=i).contiguous().pin_memory() for i in range(200)]
eng = Engine(m).prepare(xs[0])
outs = [torch.empty(eng.out_shape, pin_memory=True) for _ in xs]
for _ in range(3): eng.infer_stream(xs[:20], outs[:20])
for _ in range(3): [eng(x) for x in xs[:20]]
for r in range(3):
    t = time.perf_counter(); eng.infer_stream(xs, outs); a = (time.perf_counter() - t) / len(xs) * 1e6
    t = time.perf_counter(); [eng(x) for x in xs]; b = (time.perf_counter() - t) / len(xs) * 1e6
    print(f"per request: infer_stream {a:.1f} us ({1e6/a:.0f} img/s)  engine(x) {b:.1f} us ({1e6/b:.0f} img/s)")
