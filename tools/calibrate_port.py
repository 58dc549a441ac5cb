"""Time the oracle port (oracle/tpch.py) beside the REAL reference
(tensorquery CompiledQuery.run of the Appendix-A plans) on the same rows, one
core each -- shows the CPU baseline's "port" costs what the reference costs.
Run in the build container (the reference is importable only here):

    PYTHONPATH=/root/reference/pkg/src python tools/calibrate_port.py
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import tensorquery as ref  # noqa: E402
from tensorquery.encodings import DictionaryEncoding, EncodedTensor, StringDictionary, plain  # noqa: E402
from tensorquery.tensor import Tensor, add, mul, sub, tensor  # noqa: E402
from tensorquery.storage import FLOAT, STRING  # noqa: E402

from oracle import tpch as otpch  # noqa: E402
from paper_2211_02753_b200 import workloads as wl  # noqa: E402  (generator only)


def ref_catalog(li):
    cat = ref.Catalog()
    cols = []
    for name in wl.LINEITEM_COLUMNS:
        v = Tensor(li[name])
        if name == "l_returnflag":
            cols.append(EncodedTensor(v, DictionaryEncoding(StringDictionary(("A", "N", "R")))))
        elif name == "l_linestatus":
            cols.append(EncodedTensor(v, DictionaryEncoding(StringDictionary(("F", "O")))))
        else:
            cols.append(plain(v))
    cat.register("lineitem", ref.table_from_columns(list(wl.LINEITEM_COLUMNS), cols))
    return cat


def registries():
    def q1prep(rf, ls, q, p, d, t):
        one = tensor(1.0)
        dp = mul(p.values, sub(one, d.values))
        ch = mul(dp, add(one, t.values))
        return (rf, ls, q, p, plain(dp), plain(ch), d)

    r1 = ref.UdfRegistry()
    r1.register(ref.UdfEntry("q1prep", (("rf", STRING), ("ls", STRING), ("qty", FLOAT),
                                        ("price", FLOAT), ("disc_price", FLOAT), ("charge", FLOAT),
                                        ("disc", FLOAT)), 6, q1prep, (), pe_outputs=False))
    r6 = ref.UdfRegistry()
    r6.register(ref.UdfEntry("revenue", (("rev", FLOAT),), 2,
                             lambda p, d: (plain(mul(p.values, d.values)),), (), pe_outputs=False))
    return {"q1": (wl.Q1_SQL, r1, otpch.q1), "q6": (wl.Q6_SQL, r6, otpch.q6)}


def best_of(fn, reps=3):
    t = []
    for _ in range(reps):
        w0 = time.perf_counter()
        fn()
        t.append(time.perf_counter() - w0)
    return min(t)


def main():
    out = {}
    for rows in (1_000_000, 3_000_000):
        li = wl.lineitem_arrays(10.0, 42, rows=60_000_000, lo=0, hi=rows)
        cat = ref_catalog(li)
        for q, (sql, reg, port) in registries().items():
            cq = ref.compile_plan(ref.lower(ref.bind(ref.parse(sql), cat, reg)),
                                  ref.CompileConfig(), reg)
            res = cq.run(cat)
            exp = port(li)
            for nm, col in zip(res.schema.names, res.columns):
                np.testing.assert_allclose(col.values.data, exp[nm], rtol=1e-9)
            t_ref = best_of(lambda: cq.run(cat))
            t_port = best_of(lambda: port(li))
            out[f"{q}_{rows}"] = {"reference_rows_per_s": rows / t_ref,
                                  "port_rows_per_s": rows / t_port,
                                  "port_over_reference": t_ref / t_port}
            print(q, rows, json.dumps(out[f"{q}_{rows}"]), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
