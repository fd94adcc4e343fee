"""The C-ABI library loads on a CPU-only host and exports every symbol
include/helmgpu.h declares (no compute calls)."""

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    text = open(os.path.join(ROOT, "include", "helmgpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hg_[a-z_A-Z0-9]+)\s*\(", text)))


def test_header_declares_the_abi():
    names = _declared()
    for must in ("hg_precond_create", "hg_precond_apply", "hg_gmres", "hg_solve_host", "hg_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2406_06283_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libhelmgpu.so not built")
    lib = _lib.load()
    for name in _declared():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, name
    assert lib.hg_abi_version() == _lib.ABI_VERSION
    assert lib.hg_last_error() == b""


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2406_06283_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", src, flags=re.M), f


def test_python_constants_match_header():
    """Host arrays sized from _lib must match the header's sizes."""
    from paper_2406_06283_b200 import _lib

    text = open(os.path.join(ROOT, "include", "helmgpu.h")).read()
    consts = dict(re.findall(r"#define (HG_[A-Z0-9_]+) (\d+)", text))
    assert int(consts["HG_NPHASES"]) == _lib.NPHASES == len(_lib.PHASES)
    assert int(consts["HG_MAX_RHS"]) == _lib.MAX_RHS
    assert int(consts["HG_ABI_VERSION"]) == _lib.ABI_VERSION
    assert int(consts["HG_ORTH_MEASURED"]) == _lib.ORTH["measured"]
    assert int(consts["HG_ORTH_DCGS2"]) == _lib.ORTH["dcgs2"]


def test_elman_gamma_conventions():
    """test_wgmres.py:112-126 on the mirror's host helper (no device needed)."""
    from paper_2406_06283_b200 import elman_gamma

    assert elman_gamma(1.0, 1.0, c2_bounds="norm") == 1.0
    assert elman_gamma(1.0, 4.0, c2_bounds="norm") == 0.25
    assert elman_gamma(1.0, 4.0) == 0.5
    s, lam, theta = 0.5, 1.0, 0.01
    c1 = (1 - s) / (2 + 3 * lam**4 * theta)
    c2 = 18.0 + 8.0 * lam**3
    assert c1 == pytest.approx(0.24630541871921183, rel=1e-12) and c2 == 26.0
    assert elman_gamma(c1, c2, c2_bounds="norm") == pytest.approx(c1 / 26.0)
    with pytest.raises(ValueError):
        elman_gamma(-1.0, 2.0)
    with pytest.raises(ValueError):
        elman_gamma(1.0, 2.0, c2_bounds="bogus")


def test_envelope_fields_host():
    """The envelope part of test_wgmres.py:96-109 (wgmres._envelope)."""
    import numpy as np

    from paper_2406_06283_b200.wgmres import _envelope

    env, clamped = _envelope(0.5, 3.0, 4)
    assert env.size == 5 and env[0] == 3.0 and not clamped
    assert env[1] / env[0] == pytest.approx(np.sqrt(1 - 0.25))
    env, clamped = _envelope(1.0, 3.0, 4)
    assert clamped and np.all(env[1:] == 0.0)
    assert _envelope(None, 3.0, 4) == (None, False)
