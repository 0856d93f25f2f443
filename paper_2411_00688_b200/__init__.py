"""B200-native (sm_100a) ProxSkip / PDHGSkip TV reconstruction hot path.

Drop-in for the reference ``imgskip`` L2-L4 API (same names and signatures):
operators with matched adjoints, the warm-started FGP TV prox, problem
assembly and the ProxSkip / PDHGSkip-2 / PGD / FISTA / PDHG drivers -- all
computing through hand-written CUDA kernels in ``libpsb200.so`` (C ABI:
include/psb200.h).  There is no CPU fallback; importing without the built
library raises.
"""

from . import _lib  # noqa: F401  (fails loudly when libpsb200.so is missing)
from .batched import (BatchedTvDenoise, coin_table, run_proxskip_batched, shard_balanced,
                      shard_indices)
from .devlog import CSV_HEADER, DeviceObjective, device_objective, emit_csv
from .errors import DivergenceError, ReferenceRejectedError
from .operators import (BlurKernel, LinearMap, RadonGeometry, blur_adjoint, blur_forward, blur_map,
                        block_stack, diagonal_map, divergence, gaussian_kernel, grad_forward,
                        grad_map, identity_map, power_method, radon_map)
from .problems import (GRAD_NORM_SQ, DualRofProblem, TvReconstructionProblem, build_dual_rof,
                       build_tv_recon, build_tv_saddle_implicit, objective_tv, primal_from_dual)
from .phantoms import add_noise
from .proximal import project_ball, project_nonneg, prox_l2_fidelity, prox_zero
from .refsol import SELF_CONSISTENCY_TOL, ReferenceSolution, compute_reference_solution
from .skip import (SkipConfig, bernoulli_op, optimal_probability, run_pdhgskip1, run_pdhgskip2,
                   run_proxskip)
from .solvers import (IterationLog, ProxProblem, RunRecord, SaddleProblem, SmoothProblem,
                      diagonal_steps, run_aprojgd, run_fista, run_gd, run_pdhg,
                      run_pdhg_preconditioned, run_pgd)
from .tensor import axpby, dot, norm2, rel_error
from .tv import INNER_STEP, TvProxState, dual_gap_rof, tv_prox, tv_value

__version__ = "0.1.0"
