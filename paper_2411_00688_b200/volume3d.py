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

import ctypes as C
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
    """One z-slab of a config-5 problem on the current CUDA device.

    Halo planes live in receive rings: ``rb[s]`` holds plane z0-1 of the dual
    iterate q_s (slot s % 3, channels z, y, x), ``ra[s]`` plane z0+D; the
    kernel of inner iteration ``it`` reads ring slots it % 3 (q_k) and
    (it + 2) % 3 (q_{k-1}), exactly as it reads the slab's own slots, so one
    3-channel plane per neighbour and inner iteration is exchanged (the new
    q_{it+1}), not the (q_k, q_{k-1}) pair.  ``hx`` is plane z0+D of the prox
    input, exchanged once per prox call."""

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
        ring = (3, 3) + plane
        self.rb = torch.zeros(ring, dtype=dtf, device="cuda") if self.has_below else None
        self.ra = torch.zeros(ring, dtype=dtf, device="cuda") if self.has_above else None
        self.hx = torch.zeros(plane, dtype=dtf, device="cuda") if self.has_above else None
        # local send buffers of the new edge planes (used by exchanges that copy)
        self.sb = torch.zeros((3,) + plane, dtype=dtf, device="cuda") if self.has_below else None
        self.sa = torch.zeros((3,) + plane, dtype=dtf, device="cuda") if self.has_above else None
        # direct deposit (peer exchange): (base address of the neighbour's ring,
        # bytes per ring slot) -- the edge kernel stores the new plane there
        self.out_lo = None
        self.out_hi = None
        self.stream = None  # torch.cuda.Stream of this slab's work (None: current)
        self.bad = torch.full((1,), INT32_MAX, dtype=torch.int32, device="cuda")
        self.last_weight = None
        self.prox_count = 0
        self._coin = {v: torch.tensor([v], dtype=torch.uint8, device="cuda") for v in (0, 1)}

    @property
    def plane_bytes(self):
        return self.H * self.W * self.z.element_size()

    @property
    def neighbours(self):
        return self.has_below or self.has_above

    def _st(self):
        return C.c_void_p(self.stream.cuda_stream) if self.stream is not None else L.stream()

    def _send(self, s, hi):
        out = self.out_hi if hi else self.out_lo
        if out is not None:
            return C.c_void_p(out[0] + (s % 3) * out[1])
        return L.ptr(self.sa if hi else self.sb)

    # -- compute phases (one ProxSkip outer iteration) ----------------------------
    def pre(self, k, theta, gamma, p):
        L.call("psb_proxskip_pre", L.dcode(self.dto), L.dcode(self.dtf), L.ptr(self.x),
               L.ptr(self.b), 1, L.ptr(self.h), L.ptr(self.z), 1, self.x.numel(),
               L.ptr(self._coin[int(theta)]), float(gamma), gamma - gamma / p, L.ptr(self.bad), k,
               self._st())

    def fgp_part(self, it, part, weight, rep, beta_prev):
        """Inner iteration ``it`` on a plane subset: 0 = all planes, 1 = the
        interior (no halo read: runs while the exchange is in flight), 2 = the
        two edge planes (after the halos of q_it arrived; their new q_{it+1}
        planes also go to the send buffers / the neighbours' rings)."""
        sk, sm = it % 3, (it + 2) % 3
        rb, ra = self.rb, self.ra
        lo = self._send(it + 1, False) if (part != 1 and self.has_below) else None
        hi = self._send(it + 1, True) if (part != 1 and self.has_above) else None
        L.call("psb_fgp3d_iter_part", L.dcode(self.dtf), L.ptr(self.z), L.ptr(self.q), self.D,
               self.H, self.W, self.z0, self.Dg, it, beta_prev, self.step, weight, int(rep),
               int(self.nonneg), L.ptr(rb[sk]) if rb is not None else None,
               L.ptr(rb[sm]) if rb is not None else None,
               L.ptr(ra[sk]) if ra is not None else None,
               L.ptr(ra[sm]) if ra is not None else None, L.ptr(self.hx), 0, int(part), lo, hi,
               self._st())

    def fgp_iter(self, it, weight, rep, beta_prev):
        self.fgp_part(it, 0, weight, rep, beta_prev)

    def rotate_rings(self, n):
        """Start of a prox call: q_0 is the previous call's q_n (the post kernel
        moved it to slot 0), whose halo planes are already in ring slot n % 3."""
        s = n % 3
        if s == 0:
            return
        with torch.cuda.stream(self.stream) if self.stream is not None else _nullctx():
            for r in (self.rb, self.ra):
                if r is not None:
                    r[0].copy_(r[s])

    def chain_pre(self, pend, kfirst, gamma, p):
        """Prox input after `pend` deferred skips, x left stale in memory."""
        L.call("psb_skip_chain", L.dcode(self.dto), L.dcode(self.dtf), L.ptr(self.x),
               L.ptr(self.b), L.ptr(self.h), L.ptr(self.z), self.x.numel(), int(pend),
               float(gamma), gamma - gamma / p, L.ptr(self.bad), int(kfirst), self._st())

    def flush(self, pend, kfirst, gamma):
        L.call("psb_skip_chain", L.dcode(self.dto), L.dcode(self.dtf), L.ptr(self.x),
               L.ptr(self.b), L.ptr(self.h), None, self.x.numel(), int(pend), float(gamma), 0.0,
               L.ptr(self.bad), int(kfirst), self._st())

    def post(self, k, gamma, p, pend=0):
        hqn = self.rb[self.inner % 3] if self.rb is not None else None
        L.call("psb_proxskip_post3d", L.dcode(self.dto), L.dcode(self.dtf), L.ptr(self.x),
               L.ptr(self.b), L.ptr(self.h), L.ptr(self.z), L.ptr(self.q), L.ptr(hqn),
               self.D, self.H, self.W, self.z0, self.Dg, self.inner, int(self.nonneg),
               float(gamma), p / gamma, int(pend), L.ptr(self.bad), k, self._st())

    def check_finite(self):
        kb = int(self.bad.item())
        if kb != INT32_MAX:
            raise DivergenceError(kb, "proxskip3d")


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


class LocalExchange:
    """Slabs of this process on one stream (the 1-GPU emulation of the
    decomposition).  ``direct`` (default): each edge kernel stores its new
    planes straight into the neighbours' rings (the peer-memory data path,
    with plain device pointers); otherwise the planes go through the local
    send buffers and a device copy (the NCCL data path)."""

    def __init__(self, direct=True):
        self.direct = direct

    def setup(self, slabs):
        for i, s in enumerate(slabs):
            slot = 3 * s.plane_bytes
            if self.direct:
                s.out_lo = (slabs[i - 1].ra.data_ptr(), slot) if s.has_below else None
                s.out_hi = (slabs[i + 1].rb.data_ptr(), slot) if s.has_above else None

    def begin_prox(self, slabs):
        for i, s in enumerate(slabs[:-1]):
            s.hx.copy_(slabs[i + 1].z[0])

    def wait_ring(self, slabs, m):
        pass

    def send(self, slabs, m):
        if self.direct:
            return
        for i, s in enumerate(slabs):
            if s.has_below:
                slabs[i - 1].ra[m % 3].copy_(s.sb)
            if s.has_above:
                slabs[i + 1].rb[m % 3].copy_(s.sa)

    def finish(self, slabs):
        pass

    def agree_bad(self, k):
        return k


class PeerExchange:
    """Peer-memory halo exchange with stream-ordered flags (no NCCL, no host
    synchronisation): every slab runs on its own stream; a slab's edge kernel
    stores its new q_{it+1} planes directly into the neighbours' receive rings
    (NVLink peer memory across GPUs), then the stream writes the receiver's
    flag (cuStreamWriteValue32, fenced); a receiver's stream waits on its flag
    (cuStreamWaitValue32 >= seq) before the kernel that reads the ring.

    Per prox call and direction the flag advances by n + 1: "ready" (the
    sender has rotated its rings, computed its prox input and deposited its
    bottom plane into the lower neighbour's ``hx``) and one per edge kernel.
    The waits also cover the reuse hazards: a ring slot is rewritten only
    after the receiver's kernel that last read it (its edge kernel of the
    previous inner iteration, or its post kernel) has finished.

    ``peers`` maps slab index -> {"below": (ring_ptr, flag_ptr),
    "above": (ring_ptr, flag_ptr), "hx_below": ptr} -- addresses of the
    neighbours' buffers in this process (IPC-mapped for other ranks, plain
    pointers for slabs of this process: ``PeerExchange.local(slabs)``)."""

    def __init__(self, flags, peers):
        self.flags = flags  # per slab: int32 tensor [from_below, from_above] in its own memory
        self.peers = peers
        self.seq = 0
        self.group = False  # torch.distributed group of a multi-rank run (dist())

    @classmethod
    def local(cls, slabs):
        """In-process wiring (one GPU, one stream per slab): the protocol of
        the multi-GPU run with local addresses."""
        flags = [torch.zeros(2, dtype=torch.int32, device="cuda") for _ in slabs]
        peers = []
        for i, s in enumerate(slabs):
            d = {}
            if s.has_below:
                nb = slabs[i - 1]
                d["below"] = (nb.ra.data_ptr(), flags[i - 1].data_ptr() + 4)
                d["hx_below"] = nb.hx.data_ptr()
            if s.has_above:
                na = slabs[i + 1]
                d["above"] = (na.rb.data_ptr(), flags[i + 1].data_ptr())
            peers.append(d)
        for s in slabs:
            if s.stream is None:
                s.stream = torch.cuda.Stream()
        return cls(flags, peers)

    @classmethod
    def dist(cls, slab, group=None):
        """Multi-GPU wiring, one slab per rank (rank order = z order): every
        rank exports its rings, prox-input halo plane and flags as CUDA IPC
        handles, gathers its neighbours' handles over torch.distributed and
        maps them (peer access over NVLink).  Collective: every rank of the
        group calls it.  Call ``close()`` when the run is over."""
        import torch.distributed as tdist
        rank, world = tdist.get_rank(group), tdist.get_world_size(group)
        flags = torch.zeros(2, dtype=torch.int32, device="cuda")
        torch.cuda.synchronize()  # zeroed flags before any neighbour can write them
        hsize = L.LIB.psb_ipc_handle_size()

        def export(t):
            if t is None:
                return None
            h = C.create_string_buffer(hsize)
            off = C.c_int64(0)
            L.call("psb_ipc_get_handle", L.ptr(t), h, C.byref(off))
            return (h.raw, off.value)

        mine = {"ra": export(slab.ra), "rb": export(slab.rb), "hx": export(slab.hx),
                "flags": export(flags), "z0": slab.z0, "D": slab.D}
        allh = [None] * world
        tdist.all_gather_object(allh, mine, group=group)
        opened = {}

        def imp(r, key):
            h, off = allh[r][key]
            if (r, key) not in opened:
                p = C.c_void_p()
                L.call("psb_ipc_open_handle", C.create_string_buffer(h, hsize), C.byref(p))
                opened[(r, key)] = p.value
            return opened[(r, key)] + off

        d = {}
        if slab.has_below:
            if allh[rank - 1]["z0"] + allh[rank - 1]["D"] != slab.z0:
                raise ValueError("PeerExchange.dist: ranks must own consecutive slabs in z order")
            d["below"] = (imp(rank - 1, "ra"), imp(rank - 1, "flags") + 4)
            d["hx_below"] = imp(rank - 1, "hx")
        if slab.has_above:
            d["above"] = (imp(rank + 1, "rb"), imp(rank + 1, "flags"))
        ex = cls([flags], [d])
        ex.group, ex._opened = group, opened
        tdist.barrier(group=group)
        return ex

    def close(self):
        """Unmap the neighbours' buffers (after a device synchronisation)."""
        torch.cuda.synchronize()
        for p in getattr(self, "_opened", {}).values():
            L.call("psb_ipc_close", C.c_void_p(p))
        self._opened = {}

    def setup(self, slabs):
        cur = torch.cuda.current_stream()
        for i, s in enumerate(slabs):
            slot = 3 * s.plane_bytes
            p = self.peers[i]
            s.out_lo = (p["below"][0], slot) if s.has_below else None
            s.out_hi = (p["above"][0], slot) if s.has_above else None
            if s.stream is not None:
                s.stream.wait_stream(cur)

    def _signal(self, s, i, value):
        p = self.peers[i]
        if s.has_below:
            L.call("psb_stream_write_u32", s._st(), C.c_void_p(p["below"][1]), value)
        if s.has_above:
            L.call("psb_stream_write_u32", s._st(), C.c_void_p(p["above"][1]), value)

    def _wait(self, s, i, value):
        f = self.flags[i].data_ptr()
        if s.has_below:
            L.call("psb_stream_wait_geq_u32", s._st(), C.c_void_p(f), value)
        if s.has_above:
            L.call("psb_stream_wait_geq_u32", s._st(), C.c_void_p(f + 4), value)

    def begin_prox(self, slabs):
        self.seq += 1
        for i, s in enumerate(slabs):
            if s.has_below:  # bottom plane of the prox input -> hx of the slab below
                L.call("psb_copy_async", C.c_void_p(self.peers[i]["hx_below"]), L.ptr(s.z[0]),
                       s.plane_bytes, s._st())
            self._signal(s, i, self.seq)
        for i, s in enumerate(slabs):
            self._wait(s, i, self.seq)

    def wait_ring(self, slabs, m):
        # ring slot m % 3 holds q_m once the neighbour's edge kernel of
        # iteration m-1 has run (m >= 1); slot 0 (m = 0) is local (rotate_rings)
        if m == 0:
            return
        for i, s in enumerate(slabs):
            self._wait(s, i, self.seq + m)

    def send(self, slabs, m):
        for i, s in enumerate(slabs):
            self._signal(s, i, self.seq + m)

    def finish(self, slabs):
        """End of a prox call (after the post kernels)."""
        self.seq += slabs[0].inner

    def agree_bad(self, k):
        if getattr(self, "group", False) is False:
            return k
        import torch.distributed as tdist
        t = torch.tensor([int(k)], dtype=torch.int64, device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MIN, group=self.group)
        return int(t.item())


class DistExchange:
    """Halo exchange between ranks (one slab per rank, rank order = z order)
    with torch.distributed point-to-point (NCCL over NVLink; gloo in tests).

    On CUDA tensors the transfers run on a side stream: the edge planes of
    q_{it+1} leave while the interior kernel of iteration it+1 runs, and the
    compute stream waits for the transfer only before the next edge kernel."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.comm = None

    def setup(self, slabs):
        (s,) = slabs
        if s.sb is not None and s.sb.is_cuda or s.sa is not None and s.sa.is_cuda:
            self.comm = torch.cuda.Stream()

    def _p2p(self, sends, recvs):
        d = self.dist
        ops = [d.P2POp(d.isend, t.contiguous(), peer, self.group) for t, peer in sends]
        ops += [d.P2POp(d.irecv, t, peer, self.group) for t, peer in recvs]
        if not ops:
            return
        if self.comm is None:
            for req in d.batch_isend_irecv(ops):
                req.wait()
            return
        self.comm.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.comm):
            for req in d.batch_isend_irecv(ops):
                req.wait()  # orders the comm stream after NCCL, host does not block

    def begin_prox(self, slabs):
        (s,) = slabs
        sends = [(s.z[0], self.rank - 1)] if s.has_below else []
        recvs = [(s.hx, self.rank + 1)] if s.has_above else []
        self._p2p(sends, recvs)
        self._join()

    def _join(self):
        if self.comm is not None:
            torch.cuda.current_stream().wait_stream(self.comm)

    def wait_ring(self, slabs, m):
        self._join()

    def send(self, slabs, m):
        (s,) = slabs
        sends, recvs = [], []
        if s.has_below:
            sends.append((s.sb, self.rank - 1))
            recvs.append((s.rb[m % 3], self.rank - 1))
        if s.has_above:
            sends.append((s.sa, self.rank + 1))
            recvs.append((s.ra[m % 3], self.rank + 1))
        self._p2p(sends, recvs)

    def finish(self, slabs):
        pass

    def agree_bad(self, k):
        """Global first non-finite iteration: every rank raises the same
        DivergenceError (the reference stops at the first one, solvers.py:111-113)."""
        d = self.dist
        dev = "cuda" if d.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([int(k)], dtype=torch.int64, device=dev)
        d.all_reduce(t, op=d.ReduceOp.MIN, group=self.group)
        return int(t.item())


def run_proxskip_slabs(slabs, coins, *, gamma=1.0, p=0.1, exchange=None, fgp_events=None,
                       defer_skips=True):
    """K outer ProxSkip iterations over a set of slabs (one global coin stream).

    Every FGP inner iteration of a decomposed volume is two launches per slab:
    the interior planes (no halo: overlaps the exchange of the previous
    iteration's edge planes) and then the two edge planes, whose new dual
    planes go to the neighbours (``exchange``: LocalExchange in one process,
    PeerExchange over peer memory, DistExchange over torch.distributed).  A
    slab without neighbours runs one whole-slab launch per inner iteration.

    With ``defer_skips`` (default) a skipped iteration launches nothing: the
    run of skips since the last prox call is executed in registers by the next
    prox call's pre/post kernels (psb_skip_chain / psb_proxskip_post3d with
    `pend`) or by the final flush -- the same arithmetic in the same order,
    bit-identical to one pass per skip (``defer_skips=False``), without the
    16 B/voxel HBM round trip per skipped iteration.
    ``fgp_events`` (optional list) collects (start, end) CUDA events around
    each FGP inner iteration (current stream) for roofline accounting."""
    exchange = exchange or LocalExchange()
    exchange.setup(slabs)
    s0 = slabs[0]
    split = any(s.neighbours for s in slabs)
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
        exchange.begin_prox(slabs)
        for it in range(s0.inner):
            bprev = betas[it - 1] if (s0.acc and it > 0) else 0.0
            ev = None
            if fgp_events is not None:
                ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                ev[0].record()
            if split:
                for s in slabs:
                    s.fgp_part(it, 1, weight, rep, bprev)
                exchange.wait_ring(slabs, it)
                for s in slabs:
                    s.fgp_part(it, 2, weight, rep, bprev)
                exchange.send(slabs, it + 1)
            else:
                for s in slabs:
                    s.fgp_part(it, 0, weight, rep, bprev)
            if ev is not None:
                ev[1].record()
                fgp_events.append(ev)
        if split:
            exchange.wait_ring(slabs, s0.inner)
        for s in slabs:
            s.post(k, gamma, p, pend)
            s.rotate_rings(s.inner)
            s.last_weight = weight
            s.prox_count += 1
        exchange.finish(slabs)
        pend = 0
    if pend:
        for s in slabs:
            s.flush(pend, len(coins) - pend, gamma)
    cur = torch.cuda.current_stream()
    for s in slabs:
        if s.stream is not None:
            cur.wait_stream(s.stream)
    kb = exchange.agree_bad(min(int(s.bad.item()) for s in slabs))
    if kb != INT32_MAX:
        raise DivergenceError(kb, "proxskip3d")
    return [s.x for s in slabs]


def proxskip_denoise3d(b, alpha, p, seed, iters, inner_budget=20, *, n_slabs=1, precision="fp32",
                       step=STEP_3D, defer_skips=True, exchange="direct", out=None):
    """Single-process config-5 entry point (``n_slabs`` > 1 emulates the slab
    decomposition on one GPU).  ``exchange``: "direct" (edge kernels store
    into the neighbours' rings, one stream), "copy" (send buffers + copies:
    the NCCL data path), "peer" (one stream per slab, flags in device memory:
    the multi-GPU peer-memory protocol).  Returns x in the input's currency;
    ``out`` (optional, CPU input only): a contiguous CPU tensor of b's shape
    and the state dtype that receives x (page-locked: one DMA)."""
    t = AR.to_dev(b, PRECISIONS[precision][0])
    Dg = t.shape[0]
    slabs = []
    for r in range(n_slabs):
        z0, z1 = slab_bounds(Dg, r, n_slabs)
        slabs.append(Slab3D(t[z0:z1], z0, Dg, alpha, inner_budget, precision=precision, step=step))
    if exchange == "peer":
        ex = PeerExchange.local(slabs)
    elif exchange in ("direct", "copy"):
        ex = LocalExchange(direct=exchange == "direct")
    else:
        raise ValueError(f"proxskip_denoise3d: unknown exchange {exchange!r}")
    xs = run_proxskip_slabs(slabs, SkipConfig(p, seed).coins(iters), gamma=1.0, p=p,
                            defer_skips=defer_skips, exchange=ex)
    x = xs[0] if len(xs) == 1 else torch.cat(xs, dim=0)
    if out is not None:
        if (not isinstance(out, torch.Tensor) or out.is_cuda or tuple(out.shape) != tuple(x.shape)
                or out.dtype != x.dtype or not out.is_contiguous()):
            raise ValueError("proxskip_denoise3d: out must be a contiguous CPU tensor of b's shape "
                             "and the state dtype")
        return AR.download_into(out, x), slabs
    return AR.like(x, b), slabs


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
