"""cProfile of drop-in session rounds (config C4 task set, one GPU): where
the host time of a round goes once the episode runs on the device.

    python profiles/c4_round_profile.py [rounds] [P]
"""
import cProfile
import io
import os
import pstats
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    P = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    bench._ref_import()
    import torch
    sess, _ = bench.taskset_session("b200", P, 0, 1, rounds + 4)
    for _ in range(2):
        sess.run_round()
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(rounds):
        sess.run_round()
    torch.cuda.synchronize()
    pr.disable()
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(35)
    print(s.getvalue())


if __name__ == "__main__":
    main()
