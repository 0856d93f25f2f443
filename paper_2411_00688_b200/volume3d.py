"""3-D TV denoising with ProxSkip, z-slab decomposed (BASELINE config 5).

The reference is 2-D only; config 5 restates its algorithm on a
(D, H, W) volume: identity fidelity, implicit TV prox by FGP with dual step
1/12 (||grad_3D||^2 <= 12), gamma = 1, one global Philox coin stream
(skip.py:27-28).  ``tv_prox3d`` is the single-volume prox; ``Slab3D`` owns
planes [z0, z0 + D) of a volume of depth Dg, and ``run_proxskip_slabs``
advances a set of slabs in lockstep with a halo exchange before every FGP
inner iteration:

  * each slab sends its bottom plane of (q_it, q_it-1) (6 planes of H x W) to
    the slab below it in z and its top plane to the slab above; the slab
    above also needs the bottom plane of the prox input once per prox call,
    and the final dual plane once before the fused post kernel;
  * ``LocalExchange`` moves the planes between slabs held by this process
    (device copies -- the 1-GPU emulation of the decomposition);
  * ``DistExchange`` moves them between ranks with torch.distributed P2P
    (NCCL over NVLink on the GPU box; gloo on CPU in the tests).

Because the kernel's boundary tests use global plane indices, a slab set
computes exactly the whole-volume iterate (bit-identical), which the tests
check.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _arrays as AR
from . import _lib as L
from .errors import DivergenceError
from .skip import INT32_MAX, SkipConfig, _betas
from .tv import PRECISIONS

STEP_3D = 1.0 / 12.0


def slab_bounds(Dg, rank, world):
    """Planes [z0, z1) owned by ``rank`` (contiguous, sizes differ by <= 1)."""
    base, extra = divmod(Dg, world)
    z0 = rank * base + min(rank, extra)
    return z0, z0 + base + (1 if rank < extra else 0)


class Slab3D:
    """One z-slab of a config-5 problem on the current CUDA device."""

    def __init__(self, b, z0, Dg, alpha, inner_budget=20, *, precision="fp32", accelerated=True,
                 nonneg=False, step=STEP_3D):
        dto, dtf = PRECISIONS[precision]
        self.dto, self.dtf = dto, dtf
        self.b = AR.to_dev(b, dto)
        if self.b.dim() != 3:
            raise ValueError(f"Slab3D: expected (D, H, W), got {tuple(self.b.shape)}")
        self.D, self.H, self.W = self.b.shape
        self.z0, self.Dg = z0, Dg
        if z0 < 0 or z0 + self.D > Dg:
            raise ValueError("Slab3D: slab outside the volume")
        self.alpha, self.inner, self.acc, self.nonneg, self.step = alpha, inner_budget, accelerated, nonneg, step
        self.x = torch.zeros_like(self.b)
        self.h = torch.zeros_like(self.b)
        self.z = torch.empty(self.b.shape, dtype=dtf, device="cuda")
        self.q = torch.zeros((3, 3) + tuple(self.b.shape), dtype=dtf, device="cuda")
        plane = (self.H, self.W)
        self.has_below = z0 > 0
        self.has_above = z0 + self.D < Dg
        self.hb = torch.zeros((6,) + plane, dtype=dtf, device="cuda") if self.has_below else None
        self.ha = torch.zeros((6,) + plane, dtype=dtf, device="cuda") if self.has_above else None
        self.hx = torch.zeros(plane, dtype=dtf, device="cuda") if self.has_above else None
        self.hqn = torch.zeros((3,) + plane, dtype=dtf, device="cuda") if self.has_below else None
        self.bad = torch.full((1,), INT32_MAX, dtype=torch.int32, device="cuda")
        self.last_weight = None
        self.prox_count = 0
        self._coin = {v: torch.tensor([v], dtype=torch.uint8, device="cuda") for v in (0, 1)}

    # -- data exchanged with the neighbours ------------------------------------
    def _slot(self, s):
        return self.q[s % 3]

    def edge_planes(self, it):
        """(bottom, top): this slab's first / last plane of (q_it, q_it-1), each (6, H, W)."""
        qk, qm = self._slot(it), self._slot(it + 2)
        bot = torch.cat([qk[:, 0], qm[:, 0]]) if self.has_below else None
        top = torch.cat([qk[:, -1], qm[:, -1]]) if self.has_above else None
        return bot, top

    def set_halos(self, below, above):
        if self.has_below:
            self.hb.copy_(below)
        if self.has_above:
            self.ha.copy_(above)

    def prox_input_bottom(self):
        return self.z[0] if self.has_below else None

    def set_prox_input_above(self, plane):
        if self.has_above:
            self.hx.copy_(plane)

    def final_dual_top(self):
        return self._slot(self.inner)[:, -1] if self.has_above else None

    def set_final_dual_below(self, plane):
        if self.has_below:
            self.hqn.copy_(plane)

    # -- compute phases (one ProxSkip outer iteration) ----------------------------
    def pre(self, k, theta, gamma, p):
        L.call("psb_proxskip_pre", L.dcode(self.dto), L.dcode(self.dtf), L.ptr(self.x),
               L.ptr(self.b), 1, L.ptr(self.h), L.ptr(self.z), 1, self.x.numel(),
               L.ptr(self._coin[int(theta)]), float(gamma), gamma - gamma / p, L.ptr(self.bad), k,
               L.stream())

    def fgp_iter(self, it, weight, rep, beta_prev):
        hb, ha = self.hb, self.ha
        plane = self.H * self.W
        L.call("psb_fgp3d_iter", L.dcode(self.dtf), L.ptr(self.z), L.ptr(self.q), self.D, self.H,
               self.W, self.z0, self.Dg, it, beta_prev, self.step, weight, int(rep),
               int(self.nonneg), L.ptr(hb[0:3]) if hb is not None else None,
               L.ptr(hb[3:6]) if hb is not None else None,
               L.ptr(ha[0:3]) if ha is not None else None,
               L.ptr(ha[3:6]) if ha is not None else None, L.ptr(self.hx), 0, L.stream())

    def chain_pre(self, pend, kfirst, gamma, p):
        """Prox input after `pend` deferred skips, x left stale in memory."""
        L.call("psb_skip_chain", L.dcode(self.dto), L.dcode(self.dtf), L.ptr(self.x),
               L.ptr(self.b), L.ptr(self.h), L.ptr(self.z), self.x.numel(), int(pend),
               float(gamma), gamma - gamma / p, L.ptr(self.bad), int(kfirst), L.stream())

    def flush(self, pend, kfirst, gamma):
        L.call("psb_skip_chain", L.dcode(self.dto), L.dcode(self.dtf), L.ptr(self.x),
               L.ptr(self.b), L.ptr(self.h), None, self.x.numel(), int(pend), float(gamma), 0.0,
               L.ptr(self.bad), int(kfirst), L.stream())

    def post(self, k, gamma, p, pend=0):
        L.call("psb_proxskip_post3d", L.dcode(self.dto), L.dcode(self.dtf), L.ptr(self.x),
               L.ptr(self.b), L.ptr(self.h), L.ptr(self.z), L.ptr(self.q), L.ptr(self.hqn),
               self.D, self.H, self.W, self.z0, self.Dg, self.inner, int(self.nonneg),
               float(gamma), p / gamma, int(pend), L.ptr(self.bad), k, L.stream())

    def check_finite(self):
        kb = int(self.bad.item())
        if kb != INT32_MAX:
            raise DivergenceError(kb, "proxskip3d")


class LocalExchange:
    """Halo exchange between slabs that live in this process (device copies)."""

    def halos(self, slabs, it):
        edges = [s.edge_planes(it) for s in slabs]
        for i, s in enumerate(slabs):
            below = edges[i - 1][1] if i > 0 else None
            above = edges[i + 1][0] if i + 1 < len(slabs) else None
            s.set_halos(below, above)

    def prox_input(self, slabs):
        for i, s in enumerate(slabs[:-1]):
            s.set_prox_input_above(slabs[i + 1].prox_input_bottom())

    def final_dual(self, slabs):
        for i, s in enumerate(slabs[1:], start=1):
            s.set_final_dual_below(slabs[i - 1].final_dual_top())

    def agree_bad(self, k):
        return k


class DistExchange:
    """Halo exchange between ranks (one slab per rank, rank order = z order)
    with torch.distributed point-to-point (NCCL over NVLink; gloo in tests)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def _swap(self, send_down, send_up, recv_below, recv_above):
        d = self.dist
        ops = []
        if self.rank > 0:
            ops.append(d.P2POp(d.isend, send_down.contiguous(), self.rank - 1, self.group))
            ops.append(d.P2POp(d.irecv, recv_below, self.rank - 1, self.group))
        if self.rank + 1 < self.world:
            ops.append(d.P2POp(d.isend, send_up.contiguous(), self.rank + 1, self.group))
            ops.append(d.P2POp(d.irecv, recv_above, self.rank + 1, self.group))
        if ops:
            for req in d.batch_isend_irecv(ops):
                req.wait()

    def halos(self, slabs, it):
        (s,) = slabs
        bot, top = s.edge_planes(it)
        self._swap(bot, top, s.hb, s.ha)

    def prox_input(self, slabs):
        (s,) = slabs
        d = self.dist
        ops = []
        if s.has_below:
            ops.append(d.P2POp(d.isend, s.prox_input_bottom().contiguous(), self.rank - 1, self.group))
        if s.has_above:
            ops.append(d.P2POp(d.irecv, s.hx, self.rank + 1, self.group))
        if ops:
            for req in d.batch_isend_irecv(ops):
                req.wait()

    def agree_bad(self, k):
        """Global first non-finite iteration: every rank raises the same
        DivergenceError (the reference stops at the first one, solvers.py:111-113)."""
        d = self.dist
        dev = "cuda" if d.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([int(k)], dtype=torch.int64, device=dev)
        d.all_reduce(t, op=d.ReduceOp.MIN, group=self.group)
        return int(t.item())

    def final_dual(self, slabs):
        (s,) = slabs
        d = self.dist
        ops = []
        if s.has_above:
            ops.append(d.P2POp(d.isend, s.final_dual_top().contiguous(), self.rank + 1, self.group))
        if s.has_below:
            ops.append(d.P2POp(d.irecv, s.hqn, self.rank - 1, self.group))
        if ops:
            for req in d.batch_isend_irecv(ops):
                req.wait()


def run_proxskip_slabs(slabs, coins, *, gamma=1.0, p=0.1, exchange=None, fgp_events=None,
                       defer_skips=True):
    """K outer ProxSkip iterations over a set of slabs (one global coin stream).

    With ``defer_skips`` (default) a skipped iteration launches nothing: the
    run of skips since the last prox call is executed in registers by the next
    prox call's pre/post kernels (psb_skip_chain / psb_proxskip_post3d with
    `pend`) or by the final flush -- the same arithmetic in the same order,
    bit-identical to one pass per skip (``defer_skips=False``), without the
    16 B/voxel HBM round trip per skipped iteration.
    ``fgp_events`` (optional list) collects (start, end) CUDA events around
    each FGP inner-iteration launch for roofline accounting."""
    exchange = exchange or LocalExchange()
    s0 = slabs[0]
    alpha = s0.alpha
    weight = (gamma / p) * alpha  # prox_g(z, gamma/p) -> tv_prox(z, step * alpha)
    betas = _betas(s0.inner)
    pend = 0
    coins = np.asarray(coins, dtype=np.uint8)
    for k, theta in enumerate(coins):
        if defer_skips:
            if not theta:
                pend += 1
                continue
            for s in slabs:
                s.chain_pre(pend, k - pend, gamma, p)
        else:
            for s in slabs:
                s.pre(k, int(theta), gamma, p)
            if not theta:
                continue
        rep = s0.last_weight is not None and s0.last_weight != weight
        exchange.prox_input(slabs)
        for it in range(s0.inner):
            exchange.halos(slabs, it)
            bprev = betas[it - 1] if (s0.acc and it > 0) else 0.0
            ev = None
            if fgp_events is not None:
                ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                ev[0].record()
            for s in slabs:
                s.fgp_iter(it, weight, rep, bprev)
            if ev is not None:
                ev[1].record()
                fgp_events.append(ev)
        exchange.final_dual(slabs)
        for s in slabs:
            s.post(k, gamma, p, pend)
            s.last_weight = weight
            s.prox_count += 1
        pend = 0
    if pend:
        for s in slabs:
            s.flush(pend, len(coins) - pend, gamma)
    kb = exchange.agree_bad(min(int(s.bad.item()) for s in slabs))
    if kb != INT32_MAX:
        raise DivergenceError(kb, "proxskip3d")
    return [s.x for s in slabs]


def proxskip_denoise3d(b, alpha, p, seed, iters, inner_budget=20, *, n_slabs=1, precision="fp32",
                       step=STEP_3D, defer_skips=True):
    """Single-process config-5 entry point (``n_slabs`` > 1 emulates the slab
    decomposition on one GPU).  Returns x in the input's currency."""
    t = AR.to_dev(b, PRECISIONS[precision][0])
    Dg = t.shape[0]
    slabs = []
    for r in range(n_slabs):
        z0, z1 = slab_bounds(Dg, r, n_slabs)
        slabs.append(Slab3D(t[z0:z1], z0, Dg, alpha, inner_budget, precision=precision, step=step))
    xs = run_proxskip_slabs(slabs, SkipConfig(p, seed).coins(iters), gamma=1.0, p=p,
                            defer_skips=defer_skips)
    return AR.like(torch.cat(xs, dim=0), b), slabs


class TvProxState3D:
    """Warm start of the 3-D prox (the tv.py:25-50 state in 3-D)."""

    def __init__(self, shape, inner_iters, nonneg=False, dtype=torch.float32, step=STEP_3D):
        if inner_iters < 1:
            raise ValueError("TvProxState3D: inner_iters must be >= 1")
        self.slots = torch.zeros((3, 3) + tuple(shape), dtype=dtype, device="cuda")
        self.inner_iters, self.nonneg, self.step = inner_iters, nonneg, step
        self.last_weight = None
        self.total_inner_iterations = 0

    @property
    def q_warm(self):
        return AR.to_host(self.slots[0])


def tv_prox3d(x, weight, state):
    """3-D analogue of tv_prox (tv.py:53-89): u = clamp(x + div q), q warm-started."""
    if weight <= 0:
        raise ValueError(f"tv_prox3d: weight must be positive, got {weight}")
    dt = state.slots.dtype
    xd = AR.to_dev(x, dt)
    D, H, W = xd.shape
    rep = int(state.last_weight is not None and state.last_weight != weight)
    betas = _betas(state.inner_iters)
    for it in range(state.inner_iters):
        bprev = betas[it - 1] if it > 0 else 0.0
        L.call("psb_fgp3d_iter", L.dcode(dt), L.ptr(xd), L.ptr(state.slots), D, H, W, 0, D, it,
               bprev, state.step, float(weight), rep, int(state.nonneg), None, None, None, None,
               None, 0, L.stream())
    # finalize (tv.py:86-89) with the fused post kernel on a zero outer state
    # (x = b = h = 0, gamma = p = 1): it writes u = clamp(x_in + div q_n) into
    # `u` and moves q_n to slot 0.
    u = torch.zeros_like(xd)
    h = torch.zeros_like(xd)
    L.call("psb_proxskip_post3d", L.dcode(dt), L.dcode(dt), L.ptr(u), L.ptr(u), L.ptr(h), L.ptr(xd),
           L.ptr(state.slots), None, D, H, W, 0, D, state.inner_iters, int(state.nonneg), 1.0, 1.0,
           0, None, 0, L.stream())
    state.last_weight = weight
    state.total_inner_iterations += state.inner_iters
    return AR.like(u, x)
