"""B200-native HADIS cascade profiling + allocation search (arxiv 2509.00642).

Drop-in for the hot path of the reference package ``cascadesim`` 0.1.0:
``profiler.profile_config`` (grid evaluator + Pareto extractor),
``catalog.pareto_prune``, ``planner.solve`` (allocation search) and the
cascade-depth analysis ``frontier.frontier_compare``.  The
compute runs in ``libhadis_b200.so`` (hand-written sm_100a CUDA, C ABI in
``include/hadis_b200.h``); this package is the host-side mirror of the
reference's Python interface for that path.
"""

__version__ = "0.1.0"

from .catalog import (Catalog, CatalogError, ModelVariant, batch_latency,  # noqa: F401
                      default_catalog, load_catalog, make_variant, pareto_prune,
                      scaled_batch_profile, select_candidates)
from .frontier import (FrontierError, FrontierPoint, FrontierReport,  # noqa: F401
                       frontier_compare, lower_envelope, three_stage_points, two_stage_points)
from .planner import (Plan, PlannerError, brute_force_solve, fallback_plan, solve,  # noqa: F401
                      solve_many, validate_plan)
from .profiler import (THRESHOLD_GRID, CascadeRow, CascadeTable, GridProfiler,  # noqa: F401
                       ProfileError, TableProvenance, load_table, profile_config,
                       profile_records, prompts_hash, save_table)
