"""Drop-in for the reference's own driver (cli.run_single, cli.py:279-307).

``cli.run_single`` imports ``factorize`` and ``weighted_gmres`` at module
level (cli.py:31-32) and runs

    precond = factorize(forms, dec, coarse)                       # cli.py:280
    op = lambda v: precond.apply(forms.helmholtz @ v)             # cli.py:298
    rhs_p = precond.apply(rhs_vec)                                # cli.py:299
    x, rep = weighted_gmres(op, rhs_p, weight=forms.dk, ...)      # cli.py:303

``patch_helmdd()`` swaps the two names in ``helmdd.cli`` for this package's
GPU versions, so the unmodified driver runs its solve on the device.  The
host lambda of cli.py:298 is recognised, not executed per iteration:
``weighted_gmres_dropin`` finds the TwoLevelPreconditioner the lambda closes
over, checks on a seeded vector that the lambda IS M^{-1} B (its device
operator ``as_operator("T")`` must agree to 1e-12), and then runs the whole
GMRES on the device with that operator.  Any other host callable still
raises TypeError — there is no CPU fallback.
"""

import numpy as np

from .schwarz import CsrOperator, DeviceOperator, TwoLevelPreconditioner, factorize
from .wgmres import weighted_gmres

PROBE_RTOL = 1e-12


def _closure_objects(fn):
    cells = getattr(fn, "__closure__", None) or ()
    out = []
    for c in cells:
        try:
            out.append(c.cell_contents)
        except ValueError:  # empty cell
            continue
    return out


def device_operator_for(op, probe=True):
    """The device operator equivalent to ``op``: ``op`` itself when it is one,
    the preconditioned operator M^{-1} B of the TwoLevelPreconditioner a host
    lambda closes over when the lambda is that operator (checked on a seeded
    vector), else TypeError."""
    if isinstance(op, (DeviceOperator, CsrOperator)) or not callable(op):
        return op
    for obj in _closure_objects(op):
        if isinstance(obj, TwoLevelPreconditioner):
            cand = obj.as_operator("T")
            if probe:
                v = np.random.default_rng(2406).standard_normal(obj.n)
                want = np.asarray(op(v), dtype=float)
                got = cand(v)
                err = float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-300))
                if err > PROBE_RTOL:
                    continue
            return cand
    raise TypeError(
        "weighted_gmres on the GPU needs a device operator: a host callable is accepted only when it is "
        "v -> precond.apply(B @ v) for a paper_2406_06283_b200 TwoLevelPreconditioner (cli.py:298)"
    )


def weighted_gmres_dropin(op, rhs, weight=None, rtol=1e-6, maxit=200, x0=None, gamma=None):
    """wgmres.weighted_gmres's signature (wgmres.py:74), host lambda of
    cli.py:298 accepted (device_operator_for)."""
    return weighted_gmres(device_operator_for(op), rhs, weight=weight, rtol=rtol, maxit=maxit, x0=x0, gamma=gamma)


def patch_helmdd(cli_module=None):
    """Point ``helmdd.cli``'s factorize / weighted_gmres at the GPU versions.
    Returns a function that undoes the patch."""
    if cli_module is None:
        import helmdd.cli as cli_module  # noqa: PLC0415 (the reference package, when installed)
    saved = (cli_module.factorize, cli_module.weighted_gmres)
    cli_module.factorize = factorize
    cli_module.weighted_gmres = weighted_gmres_dropin

    def restore():
        cli_module.factorize, cli_module.weighted_gmres = saved

    return restore
