"""CPU oracle for the HADIS cascade-profiling + allocation hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2509_00642_b200`` imports this
package; only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline``
/ ``--impl reference`` legs of ``bench.py`` may use it, and only as the checker
or the timed CPU baseline -- never as the product path.

What it restates (reference = ``/root/reference/pkg/src/cascadesim``):

* ``grid.py``    -- record prep, grid evaluator, Pareto extractor and merge of
  ``profiler.profile_config`` (profiler.py:123-174) and
  ``catalog.pareto_prune`` (catalog.py:171-192), plus an emulation of numpy's
  pairwise float64 summation that ``np.where(...).mean()`` performs.
* ``planner.py`` -- ``planner.solve`` / ``_solve_over_rows`` / ``_evaluate_row``
  / ``fallback_plan`` / ``brute_force_solve`` / ``validate_plan``
  (planner.py:81-321).

Parity pinning: ``tests/golden/make_golden.py`` imports the genuine reference
(only possible in the build container, where ``/root/reference`` exists) and
writes golden fixtures under ``tests/golden/``; ``tests/test_oracle_golden.py``
checks this oracle against every fixture, so the oracle is pinned to the
reference's own outputs, not just to itself.
"""
