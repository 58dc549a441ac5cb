"""Dump the NVRTC source the fused scan generates for a Q1-shaped program over
compact columns (no GPU needed: tdp_pipeline_codegen never dereferences the
column pointers) and compile it with nvcc for register / spill counts.

usage: python tools/codegen_dump.py [out.cu]   (then nvcc -Xptxas -v on it)
"""

import ctypes
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2211_02753_b200 import _native as nat  # noqa: E402


def q1_compact_spec(n=60_000_000):
    fake = ctypes.c_void_p(1 << 20)  # 16-byte aligned, never dereferenced
    dts = [nat.I16, nat.U8, nat.U8, nat.I8, nat.I32, nat.I8, nat.I8]  # date rf ls qty price disc tax
    cols = nat.struct_array(nat.Column, [nat.Column(fake, d, 0, n, 1) for d in dts])
    preds = nat.struct_array(nat.Predicate, [nat.Predicate(0, nat.CMP_OPS["<="], nat.CMP_I64, 0,
                                                           10471, 0.0)])
    I = nat.Instr
    prog = [
        I(nat.OP_LOAD, nat.I64, 1, 0, 0, 0.0),            # 0 rf
        I(nat.OP_LOAD, nat.I64, 2, 0, 0, 0.0),            # 1 ls
        I(nat.OP_LOAD, nat.I64, 3, 1, 1, 50.0),           # 2 qty int [1, 50]
        I(nat.OP_LOAD, nat.I64, 4, 1, 90000, 10500000.0),  # 3 price cents
        I(nat.OP_LOAD, nat.I64, 5, 1, 0, 10.0),           # 4 disc %
        I(nat.OP_LOAD, nat.I64, 6, 1, 0, 8.0),            # 5 tax %
        I(nat.OP_CAST, nat.F64, 2, 0, 0, 0.0),            # 6 qty f64
        I(nat.OP_DECIMAL, nat.F64, 3, 0, 0, 100.0),       # 7 price
        I(nat.OP_DECIMAL, nat.F64, 4, 0, 0, 100.0),       # 8 disc
        I(nat.OP_DECIMAL, nat.F64, 5, 0, 0, 100.0),       # 9 tax
        I(nat.OP_CONST, nat.F64, 0, 0, 0, 1.0),           # 10 one
        I(nat.OP_SUB, nat.F64, 10, 8, 0, 0.0),            # 11 1-disc
        I(nat.OP_MUL, nat.F64, 7, 11, 0, 0.0),            # 12 disc_price
        I(nat.OP_ADD, nat.F64, 10, 9, 0, 0.0),            # 13 1+tax
        I(nat.OP_MUL, nat.F64, 12, 13, 0, 0.0),           # 14 charge
    ]
    prog = nat.struct_array(nat.Instr, prog)
    keys = nat.struct_array(nat.Key, [nat.Key(0, 0, 0, 3), nat.Key(1, 0, 0, 2)])
    aggs = nat.struct_array(nat.Agg, [nat.Agg(nat.AGG_COUNT, 0)] + [
        nat.Agg(nat.AGG_SUM_F64, v) for v in (6, 7, 12, 14, 8)])
    return cols, 7, n, preds, 1, prog, 15, keys, 2, aggs, 6


def main():
    out = Path(sys.argv[1] if len(sys.argv) > 1 else "/tmp/tdp_q1_compact.cu")
    lib = nat.load()
    cap = 1 << 20
    buf = ctypes.create_string_buffer(cap)
    args = q1_compact_spec()
    rc = lib.tdp_pipeline_codegen(*args, None, 0, 0, buf, cap)
    if rc < 0:
        raise SystemExit(f"codegen failed: {lib.tdp_last_error().decode()}")
    out.write_text(buf.value.decode())
    print(f"wrote {out} ({rc} bytes)")
    r = subprocess.run(["nvcc", "-cubin", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                        "-Xptxas", "-v", "-o", str(out.with_suffix(".cubin")), str(out)],
                       capture_output=True, text=True)
    print(r.stdout + r.stderr)


if __name__ == "__main__":
    main()
