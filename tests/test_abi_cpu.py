"""CPU: the C ABI's error convention (include/tdp_kernels.h) without a GPU.

Every entry point validates its descriptors before touching the device and
returns a negative status with a message in tdp_last_error() (the
reference's KernelError / ValueError discipline: validate, then raise before
computing).  These calls never launch anything, so they run on the build host.
"""

from __future__ import annotations

from ctypes import addressof, byref, c_double, c_int64, c_void_p, create_string_buffer

import pytest

from paper_2211_02753_b200 import _native as nat

EINVAL, ENOTSUP = -1, -4


@pytest.fixture(scope="module")
def lib():
    return nat.load()


def _err(lib) -> str:
    return nat.last_error()


def test_join_mode_and_negative_sizes_rejected(lib):
    info = (c_int64 * 2)()
    cols = (nat.Column * 1)()
    preds = (nat.Predicate * 1)()
    rc = lib.tdp_join_prepare_ex(None, 10, cols, 0, preds, 0, None, 10, cols, 0, preds, 0, 7,
                                 info, None, 1 << 20, None)
    assert rc == EINVAL and "mode" in _err(lib)
    rc = lib.tdp_join_prepare_ex(None, -1, cols, 0, preds, 0, None, 10, cols, 0, preds, 0, 0,
                                 info, None, 1 << 20, None)
    assert rc == EINVAL and "negative" in _err(lib)


def test_topk_bounds(lib):
    col = nat.Column(None, nat.I64, 0, 100, 1)
    out = (c_int64 * 4)()
    rc = lib.tdp_topk_order(byref(col), 0, 100, 0, out, None, 0, None)
    assert rc == EINVAL and "top-k" in _err(lib)
    rc = lib.tdp_topk_order(byref(col), 0, 100, 5000, out, None, 0, None)
    assert rc == EINVAL and "1024" in _err(lib)
    bad = nat.Column(None, nat.U8, 0, 100, 1)
    rc = lib.tdp_topk_order(byref(bad), 0, 100, 3, out, None, 0, None)
    assert rc == EINVAL and "dtype" in _err(lib)


def test_pipeline_rejects_malformed_programs(lib):
    cols = nat.columns([], device_check=False)
    # an instruction referring to a later value
    prog = nat.struct_array(nat.Instr, [nat.Instr(nat.OP_ADD, nat.F64, 1, 0, 0, 0.0)])
    buf = create_string_buffer(64)
    rc = lib.tdp_pipeline_codegen(cols, 0, 0, nat.struct_array(nat.Predicate, []), 0, prog, 1,
                                  nat.struct_array(nat.Key, []), 0,
                                  nat.struct_array(nat.Agg, []), 0, None, 0, 0, buf, 64)
    assert rc == EINVAL and "operand" in _err(lib)
    # a decimal decode must read an int64 value and have a positive divisor
    prog = nat.struct_array(nat.Instr, [nat.Instr(nat.OP_CONST, nat.F64, 0, 0, 0, 1.5),
                                        nat.Instr(nat.OP_DECIMAL, nat.F64, 0, 0, 0, 100.0)])
    rc = lib.tdp_pipeline_codegen(cols, 0, 0, nat.struct_array(nat.Predicate, []), 0, prog, 2,
                                  nat.struct_array(nat.Key, []), 0,
                                  nat.struct_array(nat.Agg, []), 0, None, 0, 0, buf, 64)
    assert rc == EINVAL and "decimal" in _err(lib)


def test_decimal_predicate_needs_integer_column_and_divisor(lib):
    host = (c_double * 10)()  # never dereferenced: validation fails first
    col = nat.Column(c_void_p(addressof(host)), nat.F64, 0, 10, 1)
    pred = nat.Predicate(0, nat.CMP_OPS["<"], nat.CMP_DEC, 0, 0, 0.5)
    out = (c_int64 * 10)()
    rc = lib.tdp_filter_select(byref(col), 1, byref(pred), 1, 10, out, out, None, 1 << 20, None)
    assert rc == EINVAL and "divisor" in _err(lib)
    pred = nat.Predicate(0, nat.CMP_OPS["<"], nat.CMP_DEC, 0, 100, 0.5)
    rc = lib.tdp_filter_select(byref(col), 1, byref(pred), 1, 10, out, out, None, 1 << 20, None)
    assert rc == EINVAL and "integer" in _err(lib)


def test_soft_linear_shape_limits(lib):
    assert lib.tdp_soft_linear_supported(nat.F32, 100_000, 64, 2, 2000, c_void_p(256)) == 1
    assert lib.tdp_soft_linear_supported(nat.F32, 100_000, 64, 2, 2000, c_void_p(260)) == 0  # X not 16-B aligned
    assert lib.tdp_soft_linear_supported(nat.F32, 100_000, 48, 2, 2000, c_void_p(256)) == 1  # strided
    assert lib.tdp_soft_linear_supported(nat.F32, 100_000, 50, 2, 2000, c_void_p(256)) == 0  # d % 4
    assert lib.tdp_soft_linear_supported(nat.F32, 100_000, 200, 2, 2000, c_void_p(256)) == 0  # smem
    assert lib.tdp_soft_linear_supported(nat.F32, 100_000, 64, 9, 2000, c_void_p(256)) == 0  # k > 8
    assert lib.tdp_soft_linear_supported(nat.F32, 100_000, 64, 2, 9000, c_void_p(256)) == 0  # cells
    keys = (nat.SoftKey * 2)()
    keys[0] = nat.SoftKey(None, nat.SOFT_ONEHOT, nat.I64, 10)
    keys[1] = nat.SoftKey(None, nat.SOFT_ONEHOT, nat.I64, 2)  # dense key is not dense
    out = (c_int64 * 20)()
    rc = lib.tdp_linear_argmax_count(None, nat.F32, 1000, 64, 2, None, None, keys, 2, 1, out,
                                     None)
    assert rc == EINVAL and "dense" in _err(lib)


def test_replay_log_round_trip_and_validation(lib):
    """The C-side replay log (tdp_replay_log_*): a replay-mode log reports how
    far it was consumed; bad modes and oversize expect reads are rejected."""
    assert lib.tdp_replay_log_begin(3, None, 0) == EINVAL and "mode" in _err(lib)
    vals = (c_int64 * 3)(5, 6, 7)
    assert lib.tdp_replay_log_begin(2, vals, 3) == 0
    assert lib.tdp_replay_log_size() == 0  # nothing consumed yet
    assert lib.tdp_replay_log_end(None, 0) == 0
    assert lib.tdp_replay_log_begin(1, None, 0) == 0
    assert lib.tdp_replay_log_size() == 0  # nothing recorded
    out = (c_int64 * 1)()
    assert lib.tdp_replay_log_end(out, 1) == 0
    expected = (c_int64 * 17)()
    assert lib.tdp_expect_values(c_void_p(16), 8, 17, expected, None) == EINVAL
    assert "at most 16" in _err(lib)
    assert lib.tdp_expect_values(c_void_p(16), 2, 1, expected, None) == EINVAL


def test_hostread_scopes_without_device():
    """hostread: outside a scope a read is a plain read; a recording scope
    logs reads; a replaying scope hands them back in order and rejects a
    diverging sequence before touching the device."""
    import torch

    from paper_2211_02753_b200 import hostread

    t = torch.tensor([3, 4], dtype=torch.int64)
    assert hostread.read_ints(t) == [3, 4] and not hostread.active()
    with hostread.recording() as log:
        assert hostread.active()
        assert hostread.read_int(torch.tensor([9])) == 9
        hostread.record_value(11)
    assert log.values == [[9], [11]] and log.c_values == []
    with pytest.raises(RuntimeError):
        with hostread.recording():
            with hostread.recording():
                pass
    with hostread.replaying(log) as rlog:
        with pytest.raises(hostread.ReplayMismatch):  # shape differs from the log
            hostread.read_ints(torch.tensor([1, 2]))
        rlog.pos = len(log.values)
        with pytest.raises(hostread.ReplayMismatch):  # more reads than recorded
            hostread.read_int(torch.tensor([1]))
    assert not hostread.active()
