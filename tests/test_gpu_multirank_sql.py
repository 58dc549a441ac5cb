"""GPU, 2 ranks on one device (gloo): every aggregating query of the random
SQL golden (tests/golden/sql_golden.json, the reference's own results) run
row-sharded -- each rank registers its contiguous shard of every table and
runs the query inside distributed.sharded() -- must return the reference's
full-table result on both ranks: dense partials all-reduced, high-cardinality
keys repartitioned, subqueries over replicated inner results not merged
twice, ORDER BY / LIMIT after the merge, the UDF applied per shard."""

from __future__ import annotations

import json
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

G = Path(__file__).resolve().parent / "golden"


def _port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _aggregating(sql: str) -> bool:
    head = sql.split(" FROM ")[0]
    return any(f in head for f in ("COUNT(", "SUM(", "AVG(")) or sql.count("SELECT") > 1 and \
        " GROUP BY " in sql


def _worker(rank, world, port, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    sys.path.insert(0, str(G))
    import paper_2211_02753_b200 as tq
    from paper_2211_02753_b200.distributed import shard_bounds, sharded
    from paper_2211_02753_b200.encodings import DictionaryEncoding, StringDictionary, trusted
    from sql_tables import WORDS, mix_entry, tables

    meta = json.loads((G / "sql_golden.json").read_text())
    arrays = np.load(G / "sql_golden.npz")
    cat = tq.Catalog()
    for name, cols in tables().items():
        n = len(next(iter(cols.values())))
        a, b = shard_bounds(n, rank, world)
        enc = []
        with trusted():
            for cn, v in cols.items():
                if cn == "s":
                    enc.append(tq.EncodedTensor(tq.Tensor(v[a:b]),
                                                DictionaryEncoding(StringDictionary(WORDS))))
                else:
                    enc.append(tq.plain(tq.Tensor(v[a:b])))
        cat.register(name, tq.table_from_columns(list(cols), enc))
    failures, checked = [], 0
    for qi, case in enumerate(meta["cases"]):
        if "error" in case or not _aggregating(case["sql"]):
            continue
        reg = tq.UdfRegistry()
        reg.register(mix_entry(tq))
        q = tq.compile_plan(tq.lower(tq.bind(tq.parse(case["sql"]), cat, reg)),
                            tq.CompileConfig(), reg)
        try:
            with sharded():
                out = q.run(cat)
            ok = list(out.schema.names) == case["names"] and out.row_count == case["rows"]
            for ci, col in enumerate(out.columns if ok else []):
                got, exp = col.values.numpy(), arrays[f"q{qi}/{ci}"]
                if got.shape != exp.shape or got.dtype != exp.dtype:
                    ok = False
                    break
                if exp.dtype.kind == "f":
                    nan = np.isnan(exp)
                    ok &= bool(np.array_equal(np.isnan(got), nan))
                    got, exp = got[~nan], exp[~nan]
                    if exp.dtype == np.float32:
                        ok &= bool(np.allclose(got, exp, rtol=4e-7, atol=0))
                        continue
                ok &= got.tobytes() == exp.tobytes()
        except Exception as e:  # reported below
            ok = False
            print(f"rank {rank}: {case['sql']}: {type(e).__name__}: {e}", file=sys.stderr)
        checked += 1
        if not ok:
            failures.append(case["sql"])
    result[rank] = (checked, failures)


def test_two_ranks_one_gpu_random_sql_matches_reference():
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    result = mgr.dict()
    mp.start_processes(_worker, args=(2, _port(), result), nprocs=2, join=True,
                       start_method="spawn")
    for rank in (0, 1):
        checked, failures = result[rank]
        assert checked >= 100, checked
        assert not failures, failures[:5]
