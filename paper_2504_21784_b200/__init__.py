"""B200-native (sm_100a) DG S_N transport sweep fused with the gray Second-Moment
closures of arXiv 2504.21784.  See DESIGN.md and include/sweep.h."""
from .sweep import (DETERMINISTIC, EXPORTS, FIXUP, FOLD_Z, FORCE_COMM, HALF_RANGE, SIGMA_MOMENTS, Sweep, SweepError, from_problem,  # noqa: F401
                    fp64_probe, launch_floor, load_library, nccl_unique_id, run_problem, selfcheck_solves)
