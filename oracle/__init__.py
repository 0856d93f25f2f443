"""CPU oracle for the ProxSkip / PDHGSkip TV hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2411_00688_b200`` imports this
package; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may use it, and only as the checker
or the timed CPU baseline -- never as the thing measured or shipped.

``oracle.imgskip_cpu`` is a float64 numpy restatement of the reference package
``imgskip`` (``/root/reference/pkg/src/imgskip``); every function cites the
reference file:line it restates.  It is pinned against golden vectors produced
by the reference itself (``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``,
checked by ``tests/test_oracle_golden.py``).  ``oracle.tv3d_cpu`` is the 3D
restatement the reference lacks, pinned against the reference's
2D prox on plane-constant volumes.
"""
