"""CPU oracle for the ensemble-solve hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_1705_02003_b200`` imports this
package; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it, and there only as
the checker (or as the timed CPU baseline), never as the product path.

What it is: a numpy/scipy restatement of the reference (``uqgroup``) algorithm
for the hot path named by BASELINE.json ``north_star``:

* ``field2d``  – 1D Nystrom eigenpairs, 2D separable KL mode selection and the
  coefficient formula (reference ``random_field.py:59-92,145-166,174-251``);
* ``fv2d``     – the 2D 5-point finite-volume operator on the unit square, built
  with the same shared-graph / ``AssembledEnsembleSystem`` contract as the
  reference's 3D FEM (``fem3d.py:57-175``).  The reference has no 2D operator,
  so this restatement *defines* it;
* ``pcg``      – ensemble Jacobi-PCG with per-lane convergence, freeze and
  breakdown (``ensemble.py:116-281``), SpMV through scipy ``csr_matvec`` and
  dots through ``numpy.dot`` exactly as the reference does;
* ``grouping`` – stable key sort + width-S chunking with last-group replica
  padding (``grouping.py:83-122``);
* ``driver``   – ``solve_plan`` over a grouping plan (``harness.py:399-431``).

Pinning: the generic parts (SpMV, PCG, grouping, 1D eigenpairs) are checked
bit-for-bit against the reference itself by ``tests/golden/make_golden.py``
(run in the build container where ``/root/reference`` exists) and against the
committed fixtures by ``tests/test_oracle_cpu.py`` everywhere.  The 2D operator
has no reference counterpart: its goldens come from this restatement composed
with the reference's own unchanged ``ensemble_pcg``/``group_by_key``/``HierGrid``.
"""
