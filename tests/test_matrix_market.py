"""Matrix Market ingest (§8f rank 3) against the reference's own reader
(src/matrix_market.cpp via oracle/_ref): identical CSR (duplicates summed in
input order, exact zeros dropped, symmetric storage expanded) and identical
errors, for the parallel memory-mapped parser and for the files it hands to
the stream parser (signs, inf/nan, hex, subnormals, malformed tokens)."""
import numpy as np
import pytest

from conftest import bitwise


def _write(path, header, size, entries, sep="\n", trailer=""):
    with open(path, "w") as f:
        f.write(header + "\n")
        f.write("% a comment line\n%\n")
        f.write(size + "\n")
        f.write(sep.join(entries))
        f.write(trailer)


def _same(ilug, ref, path):
    ours = ilug.Matrix.read(path).csr()
    h = ref.read(path)
    want = ref.arrays(h)
    ref.free_mat(h)
    assert np.array_equal(ours[0], want[0]) and np.array_equal(ours[1], want[1])
    assert bitwise(ours[2], want[2])
    return ours


def _errors(ilug, ref, path):
    with pytest.raises(ilug.IlugError) as e:
        ilug.Matrix.read(path)
    from oracle.oracle import RefError
    with pytest.raises(RefError) as r:
        ref.read(path)
    return e.value, str(r.value)


def _random_entries(rng, n, m, k, sym=False):
    i = rng.integers(1, n + 1, k)
    j = rng.integers(1, m + 1, k)
    if sym:
        i, j = np.maximum(i, j), np.minimum(i, j)
    v = rng.standard_normal(k) * 10.0 ** rng.integers(-30, 30, k)
    v[rng.random(k) < 0.05] = 0.0  # exact zeros (dropped unless a duplicate revives them)
    return [f"{a} {b} {float(c)!r}" for a, b, c in zip(i, j, v)]


@pytest.mark.parametrize("sym", [False, True])
@pytest.mark.parametrize("k", [1, 50, 5000])
def test_mm_random_matches_reference(ilug, ref, tmp_path, sym, k):
    rng = np.random.default_rng(k + 7 * sym)
    n = 40 if k < 5000 else 700
    entries = _random_entries(rng, n, n, k, sym)
    p = str(tmp_path / "a.mtx")
    _write(p, f"%%MatrixMarket matrix coordinate real {'symmetric' if sym else 'general'}", f"{n} {n} {k}", entries)
    _same(ilug, ref, p)


def test_mm_large_parallel_path(ilug, ref, tmp_path):
    """Enough entries for the parallel triplet assembly (>= 2^20 triplets),
    with duplicates and cancellations spread over rows."""
    rng = np.random.default_rng(11)
    n, k = 5000, 1_200_000
    entries = _random_entries(rng, n, n, k)
    entries += [entries[3], entries[3].rsplit(" ", 1)[0] + " -0.0"]
    p = str(tmp_path / "big.mtx")
    _write(p, "%%MatrixMarket matrix coordinate real general", f"{n} {n} {len(entries)}", entries)
    _same(ilug, ref, p)


def test_mm_layouts(ilug, ref, tmp_path):
    """Entries split across lines, several per line, tabs/CR, trailing tokens past nnz."""
    ent = ["1 1 4.0", "2 1 -1.5e+00", "2 2 4", "3 3 1E2", "1 3 .5", "3 1 -.25", "2 2 0.5"]
    p = str(tmp_path / "l.mtx")
    with open(p, "w") as f:
        f.write("%%MatrixMarket matrix coordinate integer general\r\n3 3 7\r\n")
        f.write("1 1\n4.0\t2 1 -1.5e+00 2 2 4\r\n3 3 1E2 1 3 .5\n3\n1\n-.25 2 2 0.5\n9 9 9 extra tokens\n")
    _same(ilug, ref, p)
    p2 = str(tmp_path / "l2.mtx")
    _write(p2, "%%MatrixMarket MATRIX Coordinate Real General", "3 4 7", ent, sep="   ")
    _same(ilug, ref, p2)


@pytest.mark.parametrize("val", ["+1.5", "inf", "-nan", "0x1p3", "1e-310", "1e400", "1.5d3", "2.", "-0"])
def test_mm_unusual_values(ilug, ref, tmp_path, val):
    """Tokens the fast parser declines go through the stream parser: the result
    or the error is the reference's."""
    p = str(tmp_path / "u.mtx")
    _write(p, "%%MatrixMarket matrix coordinate real general", "2 2 3", ["1 1 1.0", f"2 1 {val}", "2 2 3.0"])
    try:
        h = ref.read(p)
    except Exception:
        e, r = _errors(ilug, ref, p)
        assert e.message.split("'")[-1] == r.split("'")[-1]
        return
    ref.free_mat(h)
    _same(ilug, ref, p)


@pytest.mark.parametrize("body,size", [
    (["1 1 1.0", "2 2"], "2 2 2"),              # truncated
    (["1 1 1.0", "3 1 2.0"], "2 2 2"),          # row out of range
    (["1 1 1.0", "2 0 2.0", "x y z"], "2 2 3"),  # column 0 before a malformed entry
    (["1 1 1.0", "+2 1 2.0"], "2 2 2"),         # signed index (stream parser)
    (["1 1 1.0", "1.0 1 2.0"], "2 2 2"),        # non-integer index
])
def test_mm_errors_match_reference(ilug, ref, tmp_path, body, size):
    p = str(tmp_path / "e.mtx")
    _write(p, "%%MatrixMarket matrix coordinate real general", size, body)
    try:
        h = ref.read(p)
    except Exception:
        e, r = _errors(ilug, ref, p)
        assert e.status == 2  # io -> 2 at the C ABI
        assert e.message.split("'")[-1] == r.split("'")[-1], (e.message, r)
        return
    ref.free_mat(h)
    _same(ilug, ref, p)


@pytest.mark.parametrize("header", ["%%MatrixMarket matrix array real general",
                                    "%%MatrixMarket matrix coordinate complex general",
                                    "%%MatrixMarket matrix coordinate pattern general",
                                    "%%MatrixMarket matrix coordinate real hermitian",
                                    "%MatrixMarket matrix coordinate real general"])
def test_mm_header_errors(ilug, ref, tmp_path, header):
    p = str(tmp_path / "h.mtx")
    _write(p, header, "2 2 1", ["1 1 1.0"])
    e, r = _errors(ilug, ref, p)
    assert e.message.split("'")[-1] == r.split("'")[-1]


def test_mm_generated_roundtrip_matches_reference(ilug, ref, tmp_path):
    """mm_write then both readers: the C2-family operator at a small size."""
    A = ilug.Matrix.generate("pressure27(12,11,10)")
    p = str(tmp_path / "p.mtx")
    A.write(p)
    got = _same(ilug, ref, p)
    for x, y in zip(got, A.csr()):
        assert np.array_equal(x, y)


def test_mm_write_text_matches_reference(ilug, ref, tmp_path):
    """The parallel writer emits the reference writer's bytes (several row blocks)."""
    A = ilug.Matrix.generate("stencil27(48,48,40)")
    ours, theirs = str(tmp_path / "o.mtx"), str(tmp_path / "r.mtx")
    A.write(ours)
    h = ref.mat(*A.csr())
    ref.write(h, theirs)
    ref.free_mat(h)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
