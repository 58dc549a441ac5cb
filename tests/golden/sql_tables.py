"""The two tables of the random-SQL golden cases (make_sql_golden.py): the
generator and the tests rebuild them from the same seeds; the checksums in
sql_golden.json pin them."""

import numpy as np

WORDS = ("apple", "kiwi", "lemon", "pear")
INT_COLS = ("k1", "k2", "big", "r", "v")
FLOAT_COLS = ("f", "g")
# t: small; u: >= 65 536 rows (hash group-by); w: >= 148 x 2048 rows (the
# bulk-copy ring kernels; only aggregates or LIMITed rows are stored)
SIZES = {"t": (4096, 1), "u": (70_000, 2), "w": (400_000, 3)}


def make_table(n: int, seed: int) -> dict[str, np.ndarray]:
    rng = np.random.default_rng(seed)
    runs = np.repeat(np.arange(n), rng.integers(1, 6, size=n))[:n] * 7 + 100
    f = rng.integers(-200, 200, size=n) / 4.0
    f[rng.choice(n, size=3, replace=False)] = np.nan
    return {
        "k1": rng.integers(0, 7, size=n).astype(np.int64),
        "k2": rng.integers(-3, 4, size=n).astype(np.int64),
        "big": (rng.integers(0, 300, size=n) * 1_000_000_007 + 5).astype(np.int64),
        "r": runs.astype(np.int64),
        "v": rng.integers(-10**12, 10**12, size=n).astype(np.int64),
        "s": rng.integers(0, len(WORDS), size=n).astype(np.int64),
        "f": f,
        "g": (rng.integers(0, 11, size=n) / 100).astype(np.float32),
    }


def tables() -> dict[str, dict[str, np.ndarray]]:
    return {name: make_table(n, seed) for name, (n, seed) in SIZES.items()}


def mix_entry(api):
    """The UDF of the generated queries, for either implementation (`api`:
    the reference package or this one): mix(k, a, b) -> (k, x = a * 2 + b)
    -- exact in float64 for the fixture's values (multiples of 1/4)."""
    from importlib import import_module

    storage = import_module(api.__name__ + ".storage")
    tensor = import_module(api.__name__ + ".tensor")

    def body(k, a, b):
        x = tensor.add(tensor.mul(a.values, tensor.tensor(2.0)), b.values)
        return (k, api.plain(x))

    return api.UdfEntry("mix", (("k", storage.INT), ("x", storage.FLOAT)), 3, body, (),
                        pe_outputs=False)
