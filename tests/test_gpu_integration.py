"""The reference driver's solve block (cli.py:279-307) run through
patch_helmdd: a module laid out like helmdd.cli (module-level factorize /
weighted_gmres names, the cli.py:298 host lambda) is patched and its solve
block runs on the device with the reference's results (config 1 golden)."""

import types

import numpy as np
import pytest

import paper_2406_06283_b200 as hg
from paper_2406_06283_b200.integration import device_operator_for, patch_helmdd
from _helpers import golden_coarse

pytestmark = pytest.mark.gpu


def _cli_like():
    """Stand-in for helmdd.cli: the same names and the same solve block."""
    cli = types.SimpleNamespace(factorize=None, weighted_gmres=None)

    def run_solve(forms, dec, coarse, rhs_vec, rtol, maxit):
        precond = cli.factorize(forms, dec, coarse)                     # cli.py:280
        op = lambda v: precond.apply(forms.helmholtz @ v)  # noqa: E731  cli.py:298
        rhs_p = precond.apply(rhs_vec)                                  # cli.py:299
        return cli.weighted_gmres(op, rhs_p, weight=forms.dk, rtol=rtol, maxit=maxit)  # cli.py:303

    cli.run_solve = run_solve
    return cli


def test_patched_driver_solves_on_the_device(golden):
    g = golden("config1")
    P = hg.build_problem("1", workers=1, one_level=True)
    coarse = golden_coarse(g, P.forms.n_dofs)
    cli = _cli_like()
    restore = patch_helmdd(cli)
    try:
        x, rep = cli.run_solve(P.forms, P.dec, coarse, P.rhs, 1e-6, 1000)
    finally:
        restore()
    assert cli.factorize is None and cli.weighted_gmres is None  # restored
    assert rep.iterations == int(g["iterations"])
    assert np.abs(x - g["x"]).max() <= 1e-8 * np.abs(g["x"]).max()


def test_other_host_callables_are_refused(golden):
    g = golden("config1")
    P = hg.build_problem("1", workers=1, one_level=True)
    pre = hg.factorize(P.forms, P.dec, golden_coarse(g, P.forms.n_dofs))
    with pytest.raises(TypeError):
        device_operator_for(lambda v: pre.apply(v))  # M^{-1}, not M^{-1} B: the probe rejects it
    with pytest.raises(TypeError):
        device_operator_for(lambda v: 2.0 * v)
