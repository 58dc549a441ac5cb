"""Random CSV ingestion cases shared by make_csv_golden.py (runs the
reference's read_csv) and tests/test_gpu_csv_golden.py (runs this
package's): each case is a >= 64 KB file (the device tokeniser's range) of
ordinary rows with tricky cells injected -- quoting, escaped quotes,
embedded separators and newlines, whitespace, signs, exponents, inf / nan,
Python-only spellings (underscores, Unicode digits), out-of-range integers,
empty cells, short rows -- rebuilt from its seed on both sides; only the
results (column checksums, dictionaries) or the error are stored."""

from __future__ import annotations

import hashlib
import random

import numpy as np

INT_OK = ["+5", " 7 ", "-0", "1_000", "١٢٣", "-9223372036854775808", "9223372036854775807",
          "007", "-42", "  -3  ", "0", "+0"]
INT_BAD = ["0x10", "12345678901234567890", "", " ", "3.0", "1e3"]
FLOAT_OK = ["1e5", "1E-3", ".5", "5.", "inf", "-Infinity", "nan", "NaN", "1_0.5", " 3.14 ",
            "1e400", "4.9e-324", "2.2250738585072011e-308", "-0.0", "+.25",
            "1.7976931348623157e308", "0.1e-5", "12", "١.5", "-inf", "INF", "1e-400",
            "0.30000000000000004", "123456789012345678901234567890"]
FLOAT_BAD = ["0x1p3", "", "abc", "1.2.3", "--1"]
STR_TRICKS = ['"a,b"', '"say ""hi"""', '"line\nbreak"', '""', '  spaced  ', '"été"',
              '"日本"', "plain", '"x"', '"comma,and ""quote"""', " ", "tab\there"]
SHAPES = ["ints", "floats", "strs"]


def case_text(seed: int) -> tuple[str, list[tuple[str, str]]]:
    """(csv text, schema [(name, kind)]) of case `seed`."""
    rg = random.Random(seed)
    schema = [("id", "int"), ("x", "float"), ("s", "string"), ("k", "int")]
    n = 3500
    rows = []
    for i in range(n):
        x = rg.choice([f"{rg.uniform(-1e6, 1e6):.6f}", f"{rg.randint(-99, 99)}",
                       f"{rg.uniform(0, 1):.17g}", f"{rg.uniform(-1, 1):.3e}"])
        s = rg.choice(["alpha", "beta", "gamma", "delta", "eps"])
        rows.append([str(i), x, s, str(rg.randint(-10**12, 10**12))])
    tricks = rg.randint(1, 12)
    for _ in range(tricks):
        r = rg.randrange(n)
        col = rg.randrange(4)
        kind = schema[col][1]
        bad = rg.random() < 0.1
        pool = ((INT_BAD if bad else INT_OK) if kind == "int" else
                (FLOAT_BAD if bad else FLOAT_OK) if kind == "float" else STR_TRICKS)
        rows[r][col] = rg.choice(pool)
    if rg.random() < 0.05:  # a short row
        rows[rg.randrange(n)].pop()
    lines = ["id,x,s,k" if rg.random() < 0.9 else " id , x,s ,k"]
    lines += [",".join(r) for r in rows]
    end = rg.choice(["\n", "\r\n"])
    text = end.join(lines) + (end if rg.random() < 0.8 else "")
    return text, schema


def column_digest(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    if a.dtype.kind == "f":
        a = np.where(np.isnan(a), np.nan, a)  # one NaN bit pattern
    return hashlib.sha256(a.tobytes()).hexdigest()


CASES = 120
