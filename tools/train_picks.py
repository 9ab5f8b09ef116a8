import sys; sys.path.insert(0, '.')
import copy, torch
from paper_2012_02732_b200.networks import build_train_model, train_batch
from paper_2012_02732_b200.train import TrainEngine
for name in ("mobilenet_v2", "efficientnet_b0"):
    model = build_train_model(name)
    x, y = train_batch(32)
    eng = TrainEngine(copy.deepcopy(model)).prepare(x, y)
    picks = [(t.tid, eng.ops[t.tid].variant, round(eng.tuning[t.tid][0], 1)) for t in eng.prog.tasks if t.tid in eng.tuning]
    tc = [p for p in picks if p[1] >= 8000]
    print(name, "tuned", len(picks), "tcgen05", len(tc), tc[:10])
    # candidate times of a few 1x1 tasks
    eng.close()
