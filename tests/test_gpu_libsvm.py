"""Device LibSVM parser (csrc/io.cu) against the host routine (the
reference's parse_libsvm semantics, data.py:309-363): identical datasets,
identical ParseErrors (message and line), on the fast-path numbers and on
lines that fall back to the host."""

import gzip
import io

import numpy as np
import pytest

import paper_1707_06468_b200 as pb

pytestmark = pytest.mark.gpu


def _both(text, **kw):
    dev = pb.parse_libsvm(io.StringIO(text), device="auto", **kw)
    host = pb.parse_libsvm(io.StringIO(text), device=None, **kw)
    return dev, host


def _same(a, b):
    fa, fb = a.features, b.features
    assert (fa.n_rows, fa.n_cols) == (fb.n_rows, fb.n_cols)
    assert np.array_equal(fa.row_offsets, fb.row_offsets)
    assert np.array_equal(fa.col_indices, fb.col_indices)
    assert np.array_equal(fa.values.view(np.int64), fb.values.view(np.int64))  # bitwise
    assert np.array_equal(a.labels.view(np.int64), b.labels.view(np.int64))


SAMPLE = """# a comment line
1 1:0.5 3:-2   # trailing comment
-1 2:1e-3 3:4.25

+1\t1:.5 2:5. 3:-0.0
0 \x0b
7e2 10:123456789012345 11:1E+05 12:-3.14159e-7
-2.5 1:0.000001 99:22
"""


def test_fast_path_numbers_match_the_host_parser(cuda):
    dev, host = _both(SAMPLE)
    _same(dev, host)
    assert dev.features.n_cols == 99 and dev.n_samples == 6


def test_host_fallback_lines_and_crlf(cuda):
    text = ("1 1:0.30000000000000004 2:1e300\r\n"   # 17 digits, huge exponent -> host
            "1_0 2:1_5\r\n"                         # underscores: int()/float() accept them
            "2 3:0.1\r\n")
    dev, host = _both(text)
    _same(dev, host)
    for bad in ("-1 1:inf 4:2\n", "1 1:nan\n"):  # parsed on the host; non-finite values are rejected
        with pytest.raises(ValueError) as ed:
            pb.parse_libsvm(io.StringIO(bad), device="auto")
        with pytest.raises(ValueError) as eh:
            pb.parse_libsvm(io.StringIO(bad), device=None)
        assert str(ed.value) == str(eh.value)


@pytest.mark.parametrize("text,line,fragment", [
    ("1 1:0.5\nbad 1:2\n", 2, "non-numeric label"),
    ("1 1:0.5\n1 2:1 3\n", 2, "malformed feature token '3'"),
    ("1 1:0.5\n1 2:1 2:3\n", 2, "non-increasing feature index 2"),
    ("1 1:0.5\n1 0:1\n", 2, "non-increasing feature index 0"),
    ("1 1:x\n1 2:1 2:3\n", 1, "malformed feature token '1:x'"),  # host-checked line before a device error
    ("1 1:1.5.5\n", 1, "malformed feature token"),
    ("\n# only comments\n", None, "empty input"),
])
def test_errors_match_the_host_parser(cuda, text, line, fragment):
    with pytest.raises(pb.ParseError) as ed:
        pb.parse_libsvm(io.StringIO(text), device="auto")
    with pytest.raises(pb.ParseError) as eh:
        pb.parse_libsvm(io.StringIO(text), device=None)
    assert str(ed.value) == str(eh.value)
    assert ed.value.line == line and fragment in str(ed.value)


def test_n_cols_override_and_gzip(cuda, tmp_path):
    dev, host = _both("1 2:1.0\n", n_cols=5)
    _same(dev, host)
    assert dev.n_features == 5
    with pytest.raises(pb.ParseError):
        pb.parse_libsvm(io.StringIO("1 7:1.0\n"), n_cols=5, device="auto")
    data = pb.gen_sparse_glm(300, 80, 0.1, 3)
    path = tmp_path / "d.svm.gz"
    pb.to_libsvm(data, path)  # repr floats: mostly host-converted lines
    dev = pb.parse_libsvm(path, device="auto")
    host = pb.parse_libsvm(path, device=None)
    _same(dev, host)
    assert np.array_equal(dev.features.values, data.features.values)


def test_large_generated_file_round_trip(cuda):
    """A config-2-shaped file written with 6 significant digits (all on the
    device fast path) parses to exactly what the host parser returns."""
    rng = np.random.default_rng(5)
    n, p, k = 20_000, 50_000, 20
    rows = []
    for i in range(n):
        cols = np.sort(rng.choice(p, size=k, replace=False)) + 1
        vals = rng.standard_normal(k)
        rows.append(f"{rng.choice([-1, 1])} " + " ".join(f"{c}:{v:.6g}" for c, v in zip(cols, vals)))
    text = "\n".join(rows) + "\n"
    dev, host = _both(text)
    _same(dev, host)
    assert dev.features.nnz == n * k


def test_exact_conversion_of_17_digit_and_random_decimals(cuda):
    """The device's Eisel-Lemire path: repr() of random doubles over the whole
    normal range and random decimal strings of up to 19 digits parse to the
    same bits as float() (the host routine); the device handles the file
    (no host fallback decision)."""
    import struct

    from paper_1707_06468_b200 import data as D

    rng = np.random.default_rng(17)
    vals = []
    bits = rng.integers(0, 2 ** 63, size=60_000, dtype=np.int64)
    for b in bits:
        x = struct.unpack("<d", struct.pack("<q", int(b)))[0]
        if np.isfinite(x) and x != 0 and abs(x) > 2.3e-308:
            vals.append(repr(float(x)))
    for _ in range(60_000):
        nd = int(rng.integers(1, 20))
        s = "".join(str(int(c)) for c in rng.integers(0, 10, size=nd))
        pos = int(rng.integers(0, nd + 1))
        s = s[:pos] + "." + s[pos:]
        if rng.random() < 0.5:
            s += f"e{int(rng.integers(-290, 280))}"
        if s[0] == "." and len(s) == 1:
            continue
        vals.append(s if rng.random() < 0.5 else "-" + s)
    lines = []
    for i in range(0, len(vals), 20):
        chunk = vals[i:i + 20]
        lines.append("1 " + " ".join(f"{j + 1}:{v}" for j, v in enumerate(chunk)))
    text = "\n".join(lines) + "\n"
    raw = text.encode()
    dev = D._parse_device(raw, None)
    assert dev is not None  # the device path handled it
    host = pb.parse_libsvm(io.StringIO(text), device=None)
    _same(dev, host)
