"""Reference-solution generation on the device.

The reference harness computes the u* that rel_error is measured against with
long runs (harness.py:209-262): accelerated projected gradient on the dual
for the denoising experiments, diagonally preconditioned PDHG on the explicit
splitting otherwise, each with a half-budget self-consistency check
(SELF_CONSISTENCY_TOL, harness.py:42).  ``compute_reference_solution`` runs
the same algorithms with the same check through the fused native paths:

* dual ROF: ``run_aprojgd`` = one FGP burst (solvers._aprojgd_dual_fused);
  the half-budget iterate is a second, shorter burst (FISTA's momentum makes
  a run not splittable, and both bursts are deterministic);
* explicit CT: ``run_pdhg_preconditioned`` in the native PDHG driver with the
  diagonal steps; the run is split at iters // 2 and continued from (x, y),
  which is exactly one run because (x, y) is PDHG's whole state.

Other problems fall back to the reference's single observed run.  The disk
cache and config hashing of the harness are control plane and not built.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ReferenceRejectedError
from .problems import DualRofProblem, TvReconstructionProblem, primal_from_dual
from .solvers import IterationLog, diagonal_steps, run_aprojgd, run_pdhg, run_pdhg_preconditioned
from .tensor import rel_error

SELF_CONSISTENCY_TOL = 1e-6


@dataclass
class ReferenceSolution:
    u_star: np.ndarray
    provenance: dict = field(default_factory=dict)
    config_hash: str = ""


def compute_reference_solution(problem, iters, tol=SELF_CONSISTENCY_TOL):
    """Long-run u* of a dual-ROF problem (``build_dual_rof``) or of a TV
    reconstruction problem (its explicit saddle form is built if missing)."""
    if iters < 2:
        raise ValueError("compute_reference_solution: need at least 2 iterations")
    half = iters // 2
    if isinstance(problem, DualRofProblem):
        g = 1.0 / problem.smooth.lipschitz
        q_half, _ = run_aprojgd(problem.smooth, problem.projector, problem.zero_dual(), g, half)
        q_full, _ = run_aprojgd(problem.smooth, problem.projector, problem.zero_dual(), g, iters)
        u_half = primal_from_dual(q_half, problem.b)
        u_full = primal_from_dual(q_full, problem.b)
        method = "aprojgd-dual"
    elif isinstance(problem, TvReconstructionProblem):
        from .problems import build_tv_recon
        prob = problem
        if prob.saddle_problem is None:
            prob = build_tv_recon(problem.A, problem.b, problem.alpha, nonneg=problem.nonneg,
                                  splitting="explicit", precision=problem.precision)
        sp = prob.saddle_problem
        if getattr(sp, "_fused", None) is not None:
            u_half, log = run_pdhg_preconditioned(sp, half)
            sigma, tau = diagonal_steps(sp.K)
            u_full, _ = run_pdhg(sp, u_half, log.y_final, sigma, tau, iters - half)
        else:
            snap = {}

            def grab_half(record, x):
                if record.iteration == half:
                    snap["x"] = np.array(x, copy=True)

            u_full, _ = run_pdhg_preconditioned(sp, iters, IterationLog(callback=grab_half))
            u_half = snap["x"]
        method = "pdhg-preconditioned-explicit"
    else:
        raise TypeError("compute_reference_solution: expected a DualRofProblem or a "
                        "TvReconstructionProblem")
    sc = rel_error(u_half, u_full)
    if sc > tol:
        raise ReferenceRejectedError(sc, tol)
    return ReferenceSolution(u_star=np.asarray(u_full, dtype=np.float64),
                             provenance=dict(method=method, iterations=iters,
                                             self_consistency_error=sc))
