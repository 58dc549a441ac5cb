"""GPU: device CSV ingestion (csvdev.py, csrc/csv.cu).

The device path must give the host reader's table bit for bit -- the host
reader being the reference's read_csv (tq/storage.py:206-249: csv.reader,
int(), float(), dict_encode) -- and must hand every file it does not model
(stray quotes, empty lines, wrong field counts, invalid cells) to the host
reader, so errors are the reference's exactly."""

from __future__ import annotations

import io

import numpy as np
import pytest

import paper_2211_02753_b200 as tq
from paper_2211_02753_b200 import csvdev, storage

pytestmark = pytest.mark.gpu

SCHEMA = tq.Schema((("id", tq.ColumnType("int")), ("price", tq.ColumnType("float")),
                    ("flag", tq.ColumnType("string")), ("qty", tq.ColumnType("int")),
                    ("note", tq.ColumnType("string"))))


def _host(data: bytes, schema=SCHEMA):
    return storage._read_csv_host(io.StringIO(data.decode("utf-8"), newline=""), schema, "cuda",
                                  "<csv>")


def _same(a, b):
    assert a.row_count == b.row_count
    for x, y in zip(a.columns, b.columns):
        vx, vy = x.values.numpy(), y.values.numpy()
        assert vx.dtype == vy.dtype
        np.testing.assert_array_equal(vx.view(np.uint8), vy.view(np.uint8))
        if x.is_dictionary():
            assert x.encoding.dictionary.entries == y.encoding.dictionary.entries


def _rows(n, rng, tricky=False):
    flags = ["A", "N", "R", "é", "中文", ""]
    notes = ["plain", "with,comma", 'say ""hi""', "multi\nline", "  spaced  ", "😀", ""]
    out = []
    for i in range(n):
        price = f"{rng.integers(0, 10**7) / 100:.2f}"
        if tricky:
            price = rng.choice([price, f" {price} ", f'"{price}"', "1e-7", "-0.0", "inf", "-inf",
                                "nan", "-nan", "1_000.25", ".5", "5.", "0.30000000000000004",
                                "123456789012345678901234", "2.5E+3", "1e400", "4.9e-324"])
        ident = str(i)
        if tricky:
            ident = rng.choice([ident, f"+{i}", f"-{i}", f" {i}\t", f"{i}_0", "9223372036854775807",
                                "-9223372036854775808", "007"])
        flag = rng.choice(flags)
        note = rng.choice(notes)
        note = f'"{note}"' if (tricky and ("," in note or '"' in note or "\n" in note)) else \
            note.replace(",", ";").replace('""', "'").replace("\n", " ")
        out.append(f"{ident},{price},{flag},{rng.integers(-50, 50)},{note}")
    return out


@pytest.mark.parametrize("n,tricky,eol,final", [(20_000, False, "\n", True),
                                               (20_000, False, "\r\n", False),
                                               (15_000, True, "\n", True),
                                               (15_000, True, "\r\n", True),
                                               (4_000, True, "\r", False)])
def test_device_csv_equals_host_reader(n, tricky, eol, final):
    rng = np.random.default_rng(n + len(eol) + tricky)
    text = eol.join(["id,price,flag,qty,note"] + _rows(n, rng, tricky)) + (eol if final else "")
    data = text.encode("utf-8")
    assert len(data) >= csvdev.DEVICE_CSV_MIN_BYTES
    dev = csvdev.read_csv_device(data, SCHEMA, "cuda", "<csv>")
    assert dev is not None, "the device path declined a file it models"
    _same(dev, _host(data))


def test_register_csv_takes_the_device_path(tmp_path):
    rng = np.random.default_rng(3)
    p = tmp_path / "t.csv"
    p.write_text("\n".join(["id,price,flag,qty,note"] + _rows(30_000, rng)) + "\n",
                 encoding="utf-8")
    cat = tq.Catalog()
    t = cat.register_csv(str(p), "t", SCHEMA)
    assert csvdev.LAST_PATH == "device"
    _same(t, _host(p.read_bytes()))


@pytest.mark.parametrize("case", ["field_count", "empty_cell", "bad_int", "bad_float", "header",
                                  "stray_quote", "empty_line", "overflow"])
def test_device_csv_hands_errors_and_odd_files_to_the_host(case, tmp_path):
    rng = np.random.default_rng(5)
    rows = _rows(12_000, rng)
    k = 7001
    header = "id,price,flag,qty,note"
    if case == "field_count":
        rows[k] += ",extra"
    elif case == "empty_cell":
        rows[k] = "5,,A,1,x"
    elif case == "bad_int":
        rows[k] = "5x,1.0,A,1,x"
    elif case == "bad_float":
        rows[k] = "5,1.0.0,A,1,x"
    elif case == "header":
        header = "id,cost,flag,qty,note"
    elif case == "stray_quote":
        rows[k] = '5,1.0,A"B,1,x'
    elif case == "empty_line":
        rows[k] = ""
    elif case == "overflow":
        rows[k] = "99999999999999999999,1.0,A,1,x"
    data = ("\n".join([header] + rows) + "\n").encode("utf-8")
    assert csvdev.read_csv_device(data, SCHEMA, "cuda", "<csv>") is None
    p = tmp_path / "t.csv"
    p.write_bytes(data)
    try:
        expect = _host(data)
    except Exception as e:  # noqa: BLE001 - the reference's own exception
        with pytest.raises(type(e)) as got:
            tq.Catalog().register_csv(str(p), "t", SCHEMA)
        assert str(got.value).replace(str(p), "<csv>") == str(e)
        return
    _same(tq.Catalog().register_csv(str(p), "t", SCHEMA), expect)
    assert csvdev.LAST_PATH == "host"
