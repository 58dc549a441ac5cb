"""Which framework call site issues each device operation of one eager Q3
(or Q1) run: every libtdp_kernels entry point (nat.call) and every aten op
that touches a CUDA tensor, with the innermost package frame that issued it.
Diagnostic only (GPU box): python tools/trace_plan.py [q3|q1] [sf]"""

import sys
import traceback
from collections import Counter
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
from torch.utils._python_dispatch import TorchDispatchMode  # noqa: E402

from paper_2211_02753_b200 import _native as nat, workloads as wl  # noqa: E402

PKG = "paper_2211_02753_b200"
SKIP = ("aten.view", "aten._unsafe_view", "aten.alias", "aten.detach", "aten.as_strided",
        "aten.t.", "aten.expand", "aten.slice", "aten.select", "aten.unsqueeze", "aten.squeeze",
        "aten.reshape", "aten.empty", "aten.set_", "aten.lift_fresh")


def site() -> str:
    frames = [f for f in traceback.extract_stack()[:-2] if PKG in f.filename]
    return " <- ".join(f"{Path(f.filename).name}:{f.lineno} {f.name}" for f in frames[-3:][::-1]) \
        or "?"


LOG = []


class Mode(TorchDispatchMode):
    def __torch_dispatch__(self, func, types, args=(), kwargs=None):
        kwargs = kwargs or {}
        cuda = any(isinstance(a, torch.Tensor) and a.is_cuda
                   for a in list(args) + list(kwargs.values()))
        if cuda and not str(func).startswith(SKIP):
            LOG.append(("aten", str(func), site()))
        return func(*args, **kwargs)


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "q3"
    sf = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    torch.cuda.set_device(0)
    if which == "q3":
        cat = wl.q3_catalog(wl.q3_arrays(sf, seed=7))
        plan = wl.Q3Plan(cat)
        run = lambda: plan.run_eager(cat)  # noqa: E731
    else:
        import paper_2211_02753_b200 as tq

        cat = tq.Catalog()
        cat.register("lineitem", wl.lineitem_table(wl.lineitem_arrays(sf, seed=42)))
        sql, reg = (wl.Q1_SQL, wl.q1_registry()) if which == "q1" else (wl.Q6_SQL, wl.q6_registry())
        q = wl.compile_sql(sql, cat, reg)
        run = lambda: q.run(cat)  # noqa: E731
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    orig = nat.call

    def traced(name, *args):
        LOG.append(("tdp", name, site()))
        return orig(name, *args)

    nat.call = traced
    with Mode():
        run()
    nat.call = orig
    torch.cuda.synchronize()
    for kind, name, where in LOG:
        print(f"{kind:4s} {name:40s} {where}")
    print(Counter(k for k, _, _ in LOG))


if __name__ == "__main__":
    main()
