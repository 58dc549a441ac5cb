"""Golden results of trainable (soft) queries, produced by running the
REFERENCE (build container only):

    python tests/golden/make_soft_golden.py

Every query of soft_cases.QUERIES on every applicable shape: the soft
group-by / global aggregate outputs and the tape gradients of all model
parameters for a seeded random loss over the outputs.  Writes
soft_golden.npz / soft_golden.json; checked by tests/test_gpu_soft_golden.py.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

import tensorquery as ref  # noqa: E402
from soft_cases import QUERIES, SHAPES, applicable, run_case  # noqa: E402


def main() -> None:
    arrays, cases = {}, []
    for si, shape in enumerate(SHAPES):
        for qi, sql in enumerate(QUERIES):
            if not applicable(sql, shape[3]):
                continue
            tag = f"s{si}q{qi}"
            names, outs, grads = run_case(ref, sql, shape, lambda g: np.asarray(g.data))
            for j, o in enumerate(outs):
                arrays[f"{tag}/out{j}"] = o
            for pn, g in grads.items():
                arrays[f"{tag}/grad/{pn}"] = g
            cases.append({"tag": tag, "sql": sql, "shape": list(shape), "names": names,
                          "grads": sorted(grads)})
    np.savez_compressed(HERE / "soft_golden.npz", **arrays)
    (HERE / "soft_golden.json").write_text(json.dumps({"cases": cases}, indent=1))
    print(f"{len(cases)} trainable cases")


if __name__ == "__main__":
    main()
