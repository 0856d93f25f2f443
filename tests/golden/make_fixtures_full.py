"""Full-size BASELINE-config fixtures, produced by running the REFERENCE itself.

Run in the build container (where /root/reference exists), one config per
process so they can run side by side:

    python tests/golden/make_fixtures_full.py 1 2 3 4

For each config it imports ``imgskip`` from /root/reference/pkg/src
(read-only), builds the problem exactly as SURVEY §8(d) specifies (library
path, D2/D7/D8/D9/D10 decisions), runs the reference driver for the FULL
iteration count and writes ``tests/golden/ref_full_c<N>.npz`` with:

* ``x``      final iterate (float32 -- rounding 6e-8 relative, far inside the
             1e-4 rel-L2 gate),
* ``obj``    the reference objective of that iterate in float64
             (``objective_tv``, problems.py:187-192; config 3 the unguarded
             formula, D8),
* ``prox``   prox-call count, ``inner`` total FGP inner iterations,
* ``b_sum``  float64 sum / ``b_sha`` sha256 of the input, so a test that
             regenerates the input from the seeded generators proves it is
             the same input.

Config 4 stores 32 of the 4096 problems (0, 4095 and 30 spread between),
each run for the full 300 outer iterations x FGP-50 at p = 0.1.

The GPU tests (tests/test_gpu_fullsize.py) compare the production fp32 /
mixed device path with these fixtures; nothing on the GPU box reads
/root/reference.
"""

import hashlib
import multiprocessing as mp
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
C4_INDICES = [0, 4095] + [int(i) for i in np.linspace(0, 4095, 32)[1:-1]]


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def _imports():
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, ROOT)
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import imgskip as m
    from paper_2411_00688_b200 import phantoms as ph
    return m, ph


def config1():
    m, ph = _imports()
    _, b = ph.config1_data(seed=0, n=256)
    prob = m.build_tv_recon(m.identity_map(b.shape), b, 0.1, inner_budget=100)
    x, log = m.run_proxskip(prob.prox_problem, np.zeros_like(b), None, 1.0, m.SkipConfig(0.1, 0), 500)
    return dict(x=x.astype(np.float32), obj=np.float64(m.objective_tv(x, prob)),
                prox=np.int64(log.records[-1].prox_count),
                inner=np.int64(prob.tv_state.total_inner_iterations),
                b_sum=np.float64(b.sum()), b_sha=np.array(_sha(b)))


def config2():
    m, ph = _imports()
    _, b, _ = ph.config2_data(seed=0, n=512)
    A = m.blur_map(m.gaussian_kernel(9, 2.0), b.shape)
    prob = m.build_tv_recon(A, b, 0.02, inner_budget=50)
    L = prob.prox_problem.smooth.lipschitz
    x, log = m.run_proxskip(prob.prox_problem, np.zeros_like(b), None, 1.0 / L,
                            m.SkipConfig(0.2, 0), 1000)
    return dict(x=x.astype(np.float32), obj=np.float64(m.objective_tv(x, prob)), L=np.float64(L),
                prox=np.int64(log.records[-1].prox_count),
                inner=np.int64(prob.tv_state.total_inner_iterations),
                b_sum=np.float64(b.sum()), b_sha=np.array(_sha(b)))


def config3():
    m, ph = _imports()
    from imgskip.tensor import norm2
    n = 512
    geom = m.RadonGeometry(image_side=n, n_angles=60, n_bins=725)
    A = m.radon_map(geom)
    s = A.forward(ph.config3_phantom(0, n))
    b = ph.config3_noisy(s, 0)
    prob = m.build_tv_recon(A, b, 0.05, nonneg=True, splitting="explicit")
    sp = prob.saddle_problem
    st = 1.0 / np.sqrt(sp.norm_K_sq)
    y0 = np.zeros(60 * 725 + 2 * n * n)
    x, log = m.run_pdhgskip2(sp, np.zeros((n, n)), y0, None, st, st, m.SkipConfig(0.1, 0), 2000)
    obj = 0.5 * norm2(A.forward(x) - b) ** 2 + 0.05 * m.tv_value(x)
    return dict(x=x.astype(np.float32), obj=np.float64(obj), nsq=np.float64(sp.norm_K_sq),
                prox=np.int64(log.records[-1].prox_count), x_min=np.float64(x.min()),
                b_sum=np.float64(b.sum()), b_sha=np.array(_sha(b)))


def _c4_one(i):
    m, ph = _imports()
    _, b, _ = ph.config4_problem(int(i), 256)
    # the GPU batch holds b in float32 (phantoms.config4_batch): run the
    # reference on the same float32-rounded input
    b = b.astype(np.float32).astype(np.float64)
    prob = m.build_tv_recon(m.identity_map(b.shape), b, 0.1, inner_budget=50)
    x, log = m.run_proxskip(prob.prox_problem, np.zeros_like(b), None, 1.0,
                            m.SkipConfig(0.1, int(i)), 300)
    return (x.astype(np.float32), float(m.objective_tv(x, prob)), log.records[-1].prox_count,
            prob.tv_state.total_inner_iterations, _sha(b))


def config4():
    with mp.get_context("fork").Pool(min(8, os.cpu_count() or 1)) as pool:
        res = pool.map(_c4_one, C4_INDICES)
    return dict(idx=np.array(C4_INDICES, dtype=np.int64), x=np.stack([r[0] for r in res]),
                obj=np.array([r[1] for r in res]), prox=np.array([r[2] for r in res]),
                inner=np.array([r[3] for r in res]), b_sha=np.array([r[4] for r in res]))


def main(argv):
    for c in argv or ["1", "2", "3", "4"]:
        t0 = time.time()
        out = {"1": config1, "2": config2, "3": config3, "4": config4}[c]()
        path = os.path.join(HERE, f"ref_full_c{c}.npz")
        np.savez_compressed(path, **out)
        print(f"config {c}: {path} ({os.path.getsize(path) / 1e6:.2f} MB, {time.time() - t0:.1f} s)",
              flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
