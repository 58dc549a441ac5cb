#!/usr/bin/env python
"""Benchmark of the tensor-query hot path on B200.

Default workload (the BASELINE metric): TPC-H Q1 on a synthetic SF10 lineitem
table (6.0e7 rows, 4 groups x 8 aggregates incl. avg/count), written against
the reference's query API (SQL + elementwise TvfMap UDF)
and executed by this package: Filter -> TvfMap -> GroupAggregate runs as one
fused pass (tdp_scan_aggregate); a Q6 companion runs on the same table.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--query q1|q6|q3|llp|llp-dense|image] [--sf SF] [--scaling strong|weak]

One process per GPU (torchrun for N > 1).  The table is split into N
contiguous row shards ("strong" scaling: BASELINE's "row-sharded at 1/2/4/8
GPUs"); partial aggregates are merged by an NCCL all-reduce inside the query,
and the whole step (collective included) is replayed as one CUDA graph.
Rank 0 prints one JSON line; its ``parity`` checks the timed result against
the oracle over the whole table.

``--impl reference`` times the reference's algorithm on the host cores: the
numpy restatement in oracle/ (the reference is Python/numpy and cannot be
installed on the GPU host), row-sharded over all cores with multiprocessing.

Workload modules live in benchmarks/ (tpch.py, q3.py, llp.py, image.py).
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--query", choices=("q1", "q6", "q3", "llp", "llp-dense", "image"),
                    default="q1")
    ap.add_argument("--sf", type=float, default=10.0)
    ap.add_argument("--scaling", choices=("strong", "weak"), default="strong",
                    help="strong: N row shards of one SF table (BASELINE config 2); "
                         "weak: one SF shard per rank")
    ap.add_argument("--encoding", choices=("wide", "compact"), default="wide",
                    help="compact: lossless narrow column storage (SURVEY §8(f) 1)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the full-table oracle check of the timed result")
    ap.add_argument("--no-companion", action="store_true",
                    help="skip the Q6 companion measurement of the default Q1 run")
    ap.add_argument("--image-rows", type=int, default=10_000_000)
    ap.add_argument("--image-classes", type=int, default=10)
    ap.add_argument("--llp-rows", type=int, default=100_000_000)
    ap.add_argument("--llp-features", type=int, default=64)
    ap.add_argument("--llp-classes", type=int, default=1000, help="--query llp-dense: PE classes")
    return ap.parse_args()


def main():
    args = _args()
    if args.query in ("llp", "llp-dense", "image", "q3"):
        import os

        if int(os.environ.get("RANK", "0")) != 0:
            return  # single-GPU workloads: extra ranks have nothing to do
        if args.impl == "reference":
            import json

            print(json.dumps({"impl": "reference", "unavailable":
                              f"--query {args.query} has no host reference arm; its line carries "
                              f"cpu_baseline"}))
            return
        from benchmarks import image, llp, llp_dense, q3

        {"llp": llp, "llp-dense": llp_dense, "image": image, "q3": q3}[args.query].run(args)
        return
    from benchmarks import tpch

    if args.impl == "reference":
        tpch.run_reference(args)
    else:
        tpch.run_ours(args)


if __name__ == "__main__":
    main()
