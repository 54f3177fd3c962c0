"""Halo sizes of the multi-GPU V exchange (sharded.halo_plan) per workload and
world size, from gm_shard_reach of every shard computed on one GPU (no ranks;
each shard's interval is independent of the others). For DESIGN.md §5.

  python scripts/halo_sizes.py [--workloads C2b,C5,C4,C4p,C1]
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="C1,C2b,C3n,C4p,C4,C5")
    a = ap.parse_args()
    import torch  # noqa: F401

    from paper_2005_06191_b200 import gridmdp as g
    from paper_2005_06191_b200 import sharded as S
    from paper_2005_06191_b200 import workloads as W
    print("| cfg | GPUs | halo states / step | all-gather states / step | exchange | reach pass (s) |")
    print("|---|---|---|---|---|---|")
    for name in a.workloads.split(","):
        m = g.parse_config(W.WORKLOADS[name](), name)
        n_x = int(m.sizes().n_states)
        be = S.DeviceBackend(m)
        for world in (2, 4, 8):
            t = time.perf_counter()
            reach = [be.reach(*S.ShardPlan(n_x, world, r).bounds(r)) for r in range(world)]
            dt = (time.perf_counter() - t) / world
            hp = S.halo_plan(S.ShardPlan(n_x, world, 0), reach)
            print(f"| {name} | {world} | {hp.halo_states:,} | {hp.allgather_states:,} | "
                  f"{'halo p2p' if hp.halo else 'all-gather'} | {dt:.3f} |", flush=True)


if __name__ == "__main__":
    main()
