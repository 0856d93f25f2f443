"""Multi-rank paths on CPU with the gloo backend (world_size 2 and 3).

* config 4 (batched): problem sharding covers every problem exactly once and
  needs no collective on the data path;
* config 5 (z-slabs): ``DistExchange`` -- the exact halo exchange the GPU
  run uses over NCCL -- drives a slab-decomposed FGP whose per-slab compute is
  the CPU oracle; the result must equal the whole-volume oracle bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import tv3d_cpu as o3
from oracle.imgskip_cpu import fista_betas

from paper_2411_00688_b200.volume3d import DistExchange, slab_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_iter(x, qk, qm, beta, w, step=o3.STEP_3D):
    """One accelerated FGP inner iteration on a full volume (tv.py:75-80 in 3-D)."""
    y = qk if beta == 0.0 else qk + beta * (qk - qm)
    return o3.ball_project3(y + step * o3.fd_grad3(x + o3.fd_div3(y)), w)


class OracleSlab:
    """CPU stand-in for Slab3D with the same exchange interface (receive rings
    rb / ra of the neighbours' edge planes of q_s in slot s % 3, prox-input
    plane hx, send buffers sb / sa); compute by embedding the slab + halos into
    a zero volume and running the oracle, storing only the planes of the
    requested part (1 = interior, 2 = edges + send buffers), like
    psb_fgp3d_iter_part."""

    def __init__(self, x_full, z0, z1, n_inner):
        self.Dg, self.H, self.W = x_full.shape
        self.z0, self.z1, self.D = z0, z1, z1 - z0
        self.z = torch.from_numpy(x_full[z0:z1].copy())
        self.q = torch.zeros((3, 3, z1 - z0, self.H, self.W), dtype=torch.float64)
        self.has_below, self.has_above = z0 > 0, z1 < self.Dg
        plane = (self.H, self.W)
        ring = (3, 3) + plane
        self.rb = torch.zeros(ring, dtype=torch.float64) if self.has_below else None
        self.ra = torch.zeros(ring, dtype=torch.float64) if self.has_above else None
        self.hx = torch.zeros(plane, dtype=torch.float64) if self.has_above else None
        self.sb = torch.zeros((3,) + plane, dtype=torch.float64) if self.has_below else None
        self.sa = torch.zeros((3,) + plane, dtype=torch.float64) if self.has_above else None
        self.inner = n_inner

    def fgp_part(self, it, part, beta, w):
        X = np.zeros((self.Dg, self.H, self.W))
        QK = np.zeros((3, self.Dg, self.H, self.W))
        QM = np.zeros_like(QK)
        X[self.z0:self.z1] = self.z.numpy()
        QK[:, self.z0:self.z1] = self.q[it % 3].numpy()
        QM[:, self.z0:self.z1] = self.q[(it + 2) % 3].numpy()
        if part == 2 and self.has_below:
            QK[:, self.z0 - 1] = self.rb[it % 3].numpy()
            QM[:, self.z0 - 1] = self.rb[(it + 2) % 3].numpy()
        if part == 2 and self.has_above:
            QK[:, self.z1] = self.ra[it % 3].numpy()
            QM[:, self.z1] = self.ra[(it + 2) % 3].numpy()
            X[self.z1] = self.hx.numpy()
        out = torch.from_numpy(_oracle_iter(X, QK, QM, beta, w)[:, self.z0:self.z1].copy())
        planes = range(1, self.D - 1) if part == 1 else sorted({0, self.D - 1})
        for k in planes:
            self.q[(it + 1) % 3][:, k] = out[:, k]
        if part == 2:
            if self.has_below:
                self.sb.copy_(out[:, 0])
            if self.has_above:
                self.sa.copy_(out[:, -1])

    def finalize(self):
        """u = x + div q_n on the slab (the z-term below needs ring slot n % 3)."""
        Q = np.zeros((3, self.Dg, self.H, self.W))
        Q[:, self.z0:self.z1] = self.q[self.inner % 3].numpy()
        if self.has_below:
            Q[:, self.z0 - 1] = self.rb[self.inner % 3].numpy()
        return self.z.numpy() + o3.fd_div3(Q)[self.z0:self.z1]


def _worker(rank, world, port, shape, n_inner, w, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x_full = np.random.default_rng(7).standard_normal(shape)
        z0, z1 = slab_bounds(shape[0], rank, world)
        slab = OracleSlab(x_full, z0, z1, n_inner)
        ex = DistExchange()
        ex.setup([slab])
        betas = fista_betas(n_inner)
        # the schedule of run_proxskip_slabs: interior, ring wait, edges, send
        ex.begin_prox([slab])
        for it in range(n_inner):
            beta = betas[it - 1] if it > 0 else 0.0
            slab.fgp_part(it, 1, beta, w)
            ex.wait_ring([slab], it)
            slab.fgp_part(it, 2, beta, w)
            ex.send([slab], it + 1)
        ex.wait_ring([slab], n_inner)
        u = slab.finalize()
        gathered = [None] * world
        dist.all_gather_object(gathered, (z0, z1, u, slab.q[n_inner % 3].numpy()))
        if rank == 0:
            out_q.put(gathered)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 5])
def test_slab_exchange_matches_whole_volume(world):
    shape, n_inner, w = (11, 6, 9), 6, 0.3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, n_inner, w, q))
             for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x_full = np.random.default_rng(7).standard_normal(shape)
    st = o3.Fgp3State.zeros(shape, n_inner)
    u_ref = o3.fgp_prox3(x_full, w, st)
    for z0, z1, u, qn in gathered:
        np.testing.assert_array_equal(u, u_ref[z0:z1])
        np.testing.assert_array_equal(qn, st.q[:, z0:z1])


def _shard_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_00688_b200.batched import shard_indices
        mine = shard_indices(4096, rank, world)
        n = torch.tensor([len(mine)], dtype=torch.int64)
        dist.all_reduce(n)
        gathered = [None] * world
        dist.all_gather_object(gathered, mine.tolist())
        if rank == 0:
            out_q.put((int(n.item()), gathered))
    finally:
        dist.destroy_process_group()


def test_problem_sharding_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    total, parts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert total == 4096
    assert sorted(parts[0] + parts[1]) == list(range(4096))
    assert not set(parts[0]) & set(parts[1])


def _bad_worker(rank, world, port, local, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out_q.put((rank, DistExchange().agree_bad(local[rank])))
    finally:
        dist.destroy_process_group()


def test_divergence_iteration_agreed_across_ranks():
    """A non-finite iterate on one slab makes every rank report the same
    (first) iteration -- the whole-volume run's DivergenceError."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    local = [2 ** 31 - 1, 17, 9]
    procs = [ctx.Process(target=_bad_worker, args=(r, 3, port, local, q)) for r in range(3)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(3))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == {0: 9, 1: 9, 2: 9}


def test_slab_bounds():
    for Dg, world in [(1024, 8), (23, 5), (7, 7)]:
        b = [slab_bounds(Dg, r, world) for r in range(world)]
        assert b[0][0] == 0 and b[-1][1] == Dg
        assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
