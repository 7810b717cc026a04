"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the GP hot path.

Nothing in ``paper_2403_09070_b200`` may import this package.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs use it, and only as the checker or the timed CPU
baseline, never as the product path.

``oracle.port`` restates the reference ``place3d`` algorithms for the GP inner
loop (``pkg/src/place3d/{wirelength,density,gp}.py``) in numpy/scipy, each
function citing the reference file:line it follows.  It is pinned against the
reference itself by ``tests/golden/`` fixtures generated with
``tests/golden/make_golden.py`` (run in the build container, where
``/root/reference`` can be imported) and by the reference's own known-answer
tests restated in ``tests/test_oracle.py``.

``oracle.fixed`` is the bit-exact int64 fixed-point density restatement the GPU
map is compared against.
"""
