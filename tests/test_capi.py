"""CPU: the C-ABI boundary — every symbol include/*.h declares is exported,
the config registry is the reference's (same keys, same defaults, fail-fast on
unknown keys), status codes follow src/capi.cpp:31-52, and there is no CPU
compute path (a solve without a GPU fails loudly with status 2)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = []
    for h in ("iluamg_b200.h", "ilug.h"):
        with open(os.path.join(ROOT, "include", h)) as fh:
            text = fh.read()
        names += re.findall(r"ILUAMG_API\s+[\w\s\*]+?\b(\w+)\s*\(", text)
    return names


def test_all_declared_symbols_exported(ilug):
    names = declared_symbols()
    assert len(names) >= 30 + 30
    missing = [n for n in names if not hasattr(ilug.lib, n)]
    assert not missing, missing
    # the python binding table covers the whole ABI
    assert set(names) <= set(ilug.EXPORTED_SYMBOLS)


def test_reference_entry_points_all_present(ilug):
    """The 30 iluamg_* exports of the reference (src/capi.cpp:88-228)."""
    ref_names = [n for n in declared_symbols() if n.startswith("iluamg_")]
    assert len(ref_names) == 30
    for n in ref_names:
        assert hasattr(ilug.lib, n)


def _keys(text):
    out = {}
    for line in text.splitlines():
        if line.startswith("#") or "=" not in line:
            continue
        k, rest = line.split("=", 1)
        out[k.strip()] = rest.split("#", 1)[0].strip()
    return out


def test_config_registry_matches_reference(ilug, ref):
    ref.L.iluamg_config_reference.restype = C.c_char_p
    want = _keys(ref.L.iluamg_config_reference().decode())
    got = _keys(ilug.config_reference())
    assert len(want) == 42
    for k, v in want.items():
        assert got.get(k) == v, k
    assert set(got) - set(want) == {"trisolve.upper", "krylov.form_iterates", "device.graph", "device.id",
                                    "device.amg_setup"}


def test_config_fail_fast(ilug):
    cfg = ilug.Config()
    with pytest.raises(ilug.IlugError) as e:
        cfg.set("no.such.key", "1")
    assert e.value.status == 2 and "unknown key" in e.value.message
    assert cfg.get("no.such.key") is None
    assert cfg.get("krylov.restart") == "50"


def test_config_load_file(ilug, tmp_path):
    p = tmp_path / "c.cfg"
    p.write_text("# comment\nsmoother.kind = ilu   # trailing\n\ntrisolve.m_upper=7\n")
    cfg = ilug.Config().load(str(p))
    assert cfg.get("smoother.kind") == "ilu" and cfg.get("trisolve.m_upper") == "7"
    p.write_text("bogus line\n")
    with pytest.raises(ilug.IlugError) as e:
        ilug.Config().load(str(p))
    assert e.value.status == 2 and ":1:" in e.value.message


def test_generator_errors(ilug):
    for spec, code in [("poisson2d(0,3)", 2), ("nope(3)", 2), ("poisson3d(4,4)", 2)]:
        with pytest.raises(ilug.IlugError) as e:
            ilug.Matrix.generate(spec)
        assert e.value.status == code


def test_matrix_market_roundtrip(ilug, tmp_path):
    A = ilug.Matrix.generate("pressure27(4,5,3)")
    p = str(tmp_path / "a.mtx")
    A.write(p)
    B = ilug.Matrix.read(p)
    for x, y in zip(A.csr(), B.csr()):
        assert (x == y).all()


def test_from_csr_validation(ilug):
    with pytest.raises(ilug.IlugError) as e:
        ilug.Matrix.from_csr(2, 2, [0, 2, 3], [1, 0, 0], [1.0, 2.0, 3.0])  # unsorted columns
    assert e.value.status == 2


def test_no_cpu_fallback(ilug):
    """Without a CUDA device every solve-phase entry point fails loudly (status 2)."""
    if ilug.device_count() > 0:
        pytest.skip("a GPU is present")
    A = ilug.Matrix.generate("poisson2d(8,8)")
    with pytest.raises(ilug.IlugError) as e:
        ilug.run_solve(A, ilug.Config().set("smoother.kind", "ilu"))
    assert e.value.status == 2 and "no CUDA device" in e.value.message
    with pytest.raises(ilug.IlugError):
        ilug.Smoother(A, ilug.Config())
