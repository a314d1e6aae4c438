"""B200-native (sm_100a) hot path of the Staggered Batch Scheduling simulator.

See DESIGN.md.  The compute path is libsbs_b200.so (CUDA, built in-tree by
``paper_2512_16134_b200.build``); this package is the Python view of its C-ABI.
"""
from .api import (  # noqa: F401
    REFERENCE_AGG_KEYS, ConfigError, InvariantError, SbsError, Simulator, allocate_batch,
    allocate_one,
    experiment_from_config, generate_workload, lib, library_path, run_experiment,
    schedule_decode_batch, select_decode_unit,
)
