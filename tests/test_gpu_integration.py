"""GPU: the reference-side ctypes binding shown in INTEGRATION.md is real code.

The block between the ``binding:begin`` / ``binding:end`` markers is executed
as a module with LIB_PATH pointed at the in-tree library, and its
``filter_indices`` (tdp_filter_select through plain ctypes, no package code)
must return exactly the oracle's rows (tq/kernels.py:87-96 restated)."""

from __future__ import annotations

import re
import types
from pathlib import Path

import numpy as np
import pytest

from oracle import relational as orc
from paper_2211_02753_b200 import _native

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _binding():
    text = (ROOT / "INTEGRATION.md").read_text()
    block = text.split("<!-- binding:begin", 1)[1].split("<!-- binding:end", 1)[0]
    code = re.search(r"```python\n(.*?)```", block, re.S).group(1)
    code = code.replace('"/path/to/paper_2211_02753_b200/_lib/libtdp_kernels.so"',
                        repr(str(_native.library_path())))
    mod = types.ModuleType("tq_b200_binding")
    exec(compile(code, "INTEGRATION.md", "exec"), mod.__dict__)
    return mod


@pytest.mark.parametrize("n", [0, 1, 1000, 300_001])
def test_integration_binding_filter_matches_oracle(n):
    b = _binding()
    rng = np.random.default_rng(n + 1)
    ship = rng.integers(8000, 11000, size=n).astype(np.int64)
    price = np.round(rng.uniform(900, 105000, size=n), 2)
    disc = rng.integers(0, 11, size=n) / 100.0
    cols = [ship, price, disc]
    preds = [(0, ">=", 8766), (0, "<", 9131), (2, ">=", 0.05), (2, "<=", 0.07), (1, ">", 20000.5)]
    got = b.filter_indices(cols, preds)
    exp = orc.filter_indices(cols, preds)
    np.testing.assert_array_equal(got, exp)
    # an int column against a float literal compares in float64 (numpy)
    got = b.filter_indices(cols, [(0, "<", 9000.5)])
    np.testing.assert_array_equal(got, orc.filter_indices(cols, [(0, "<", 9000.5)]))


def test_integration_binding_reports_errors():
    b = _binding()
    with pytest.raises(b.KernelError):
        b.filter_indices([np.arange(10, dtype=np.int64)], [(3, "<", 5)])  # no column 3
