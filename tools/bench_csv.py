"""Device vs host CSV ingestion throughput (diagnostic line).

A synthetic lineitem-like CSV (int dates, dictionary flags, 2-decimal prices,
quantities; pandas writes it) is ingested through csvdev.read_csv_device (the
file's bytes copied to the device and parsed there, result columns in HBM)
and, on a row sample, through the host reader (the reference's algorithm);
both results are compared bit for bit on the sample."""
import io
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import pandas as pd
import torch

import paper_2211_02753_b200 as tq
from paper_2211_02753_b200 import csvdev, storage

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 6_000_000
rng = np.random.default_rng(0)
df = pd.DataFrame({
    "l_shipdate": rng.integers(8036, 10562, rows),
    "l_returnflag": rng.choice(["A", "N", "R"], rows),
    "l_linestatus": rng.choice(["F", "O"], rows),
    "l_quantity": rng.integers(1, 51, rows),
    "l_extendedprice": rng.integers(90000, 10494951, rows) / 100.0,
    "l_discount": rng.integers(0, 11, rows) / 100.0,
    "l_tax": rng.integers(0, 9, rows) / 100.0,
})
data = df.to_csv(index=False, float_format="%.2f").encode()
schema = tq.Schema((("l_shipdate", tq.ColumnType("int")), ("l_returnflag", tq.ColumnType("string")),
                    ("l_linestatus", tq.ColumnType("string")), ("l_quantity", tq.ColumnType("int")),
                    ("l_extendedprice", tq.ColumnType("float")), ("l_discount", tq.ColumnType("float")),
                    ("l_tax", tq.ColumnType("float"))))
for _ in range(2):
    t = csvdev.read_csv_device(data, schema, "cuda", "<csv>")
torch.cuda.synchronize()
reps = 5
t0 = time.perf_counter()
for _ in range(reps):
    t = csvdev.read_csv_device(data, schema, "cuda", "<csv>")
torch.cuda.synchronize()
dev_s = (time.perf_counter() - t0) / reps
# host reader (the reference's csv.reader + int/float + dict_encode) on a sample
m = min(rows, 300_000)
sample = df.iloc[:m].to_csv(index=False, float_format="%.2f").encode()
t0 = time.perf_counter()
h = storage._read_csv_host(io.StringIO(sample.decode(), newline=""), schema, "cuda", "<csv>")
host_s = time.perf_counter() - t0
d = csvdev.read_csv_device(sample, schema, "cuda", "<csv>")
same = all(np.array_equal(a.values.numpy().view(np.uint8), b.values.numpy().view(np.uint8))
           for a, b in zip(d.columns, h.columns))
print(json.dumps({
    "metric": "CSV ingestion (register_csv) throughput", "rows": rows, "bytes": len(data),
    "device_s": dev_s, "device_gbs": len(data) / dev_s / 1e9, "device_rows_per_s": rows / dev_s,
    "host_sample_rows": m, "host_rows_per_s": m / host_s, "speedup": (rows / dev_s) / (m / host_s),
    "parity_sample_bitwise": bool(same),
    "what": "csvdev.read_csv_device: H2D of the file bytes + tokenizer + per-column parse + "
            "device dict_encode, result columns in HBM; host = storage._read_csv_host (csv "
            "module + int/float + dict_encode, the reference's read_csv) on a sample"}))
