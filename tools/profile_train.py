"""Per-task device time of the training step (GPU box):

    python tools/profile_train.py [--net mobilenet_v2] [--batch 32] [--top 25]

Each task is timed alone as a graph-captured chain (engine.profile_tasks);
prints the top tasks and the time per task kind, next to the replayed step.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


from paper_2012_02732_b200.networks import build_train_model, train_batch  # noqa: E402
from paper_2012_02732_b200.train import TrainEngine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="mobilenet_v2")
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    x, y = train_batch(a.batch)
    eng = TrainEngine(build_train_model(a.net)).prepare(x, y)
    eng.load_batch_device(x, y)
    multi, _ = eng.time_replay(True, 20)
    single, _ = eng.time_replay(False, 20)
    us = eng.profile_tasks(5)
    tasks = eng.prog.tasks
    print(f"{a.net} bs{a.batch}: step multi {multi:.1f} us, single {single:.1f} us, "
          f"sum of tasks {us.sum():.1f} us over {len(tasks)} tasks")
    kinds = {}
    for t in tasks:
        k = kinds.setdefault(t.kind, [0.0, 0])
        k[0] += us[t.tid]
        k[1] += 1
    for k, (v, n) in sorted(kinds.items(), key=lambda kv: -kv[1][0]):
        print(f"  {k:14s} {n:4d} tasks {v:9.1f} us")
    order = sorted(range(len(tasks)), key=lambda i: -us[i])[: a.top]
    for i in order:
        t = tasks[i]
        d = eng.ops[i]
        print(f"  {us[i]:8.1f} us  {t.kind:13s} {t.name:28s} params {list(d.params)[:12]}")


if __name__ == "__main__":
    main()
