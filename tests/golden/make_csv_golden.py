"""Golden results of read_csv on generated CSV files (csv_cases.py), produced
by running the REFERENCE's tensorquery.storage.read_csv (build container):

    python tests/golden/make_csv_golden.py

Records per case either the columns (dtype, row count, a checksum of the
values with one NaN bit pattern, the dictionary of string columns) or the
reference's exception class and message.  Checked by
tests/test_gpu_csv_golden.py against this package's read_csv.
"""

from __future__ import annotations

import io
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

from tensorquery import storage as rs  # noqa: E402
from csv_cases import CASES, case_text, column_digest  # noqa: E402


def main() -> None:
    out = []
    for seed in range(CASES):
        text, schema = case_text(seed)
        sch = rs.Schema(tuple((n, rs.ColumnType(k)) for n, k in schema))
        case = {"seed": seed}
        try:
            t = rs.read_csv(io.StringIO(text, newline=""), sch)
            cols = []
            for c in t.columns:
                v = np.asarray(c.values.data)
                entry = {"dtype": str(v.dtype), "rows": int(v.shape[0]),
                         "digest": column_digest(v)}
                if c.is_dictionary():
                    entry["dictionary"] = list(c.encoding.dictionary.entries)
                cols.append(entry)
            case["columns"] = cols
        except Exception as e:
            case["error"] = [type(e).__name__, str(e)]
        out.append(case)
    (HERE / "csv_golden.json").write_text(json.dumps({"cases": out}, indent=1,
                                                     ensure_ascii=False))
    errs = sum("error" in c for c in out)
    print(f"{len(out)} cases: {len(out) - errs} tables, {errs} errors")


if __name__ == "__main__":
    main()
