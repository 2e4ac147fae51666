"""CPU oracle for the spaimg V-cycle hot path — TEST INFRASTRUCTURE ONLY.

Nothing in the product package (`paper_2206_05543_b200`) imports this
package.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may use it, and only as the
checker or as the timed CPU baseline, never as the thing measured or shipped.

Two restatements of the reference algorithm (reference
`pkg/src/spaimg/multigrid.py:86-227`, `pkg/src/spaimg/stencils.py:136-153`),
both following the op-order contract of SURVEY.md Appendix A:

* `oracle.numpy_oracle` — numpy restatement in float64 and float32.
* `oracle.c_oracle`     — ctypes wrapper over `oracle/spaimg_oracle.c`
  (plain C, OpenMP, `-ffp-contract=off`), used where numpy is too slow
  (full-size configs on the GPU box) and as the CPU baseline.

Pinning: both are checked against the golden vectors the reference itself
produced in the build container (`tests/golden/make_golden.py`,
`tests/golden/ops_golden.npz`, `tests/golden/histories.json`) by
`tests/test_oracle.py`; the float64 restatements must be bitwise equal to
the reference.  The float32 half has no reference counterpart (reference
`grids.py:24` coerces to float64): it is pinned only through its float64
twin (same expression trees, checked to 1e-6 relative) — "parity unpinned"
for fp32 beyond that.
"""
