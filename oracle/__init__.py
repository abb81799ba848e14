"""CPU oracle for the DPM hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker
(or the timed CPU baseline).  The product package paper_2012_08099_b200 never
imports it.  See oracle/dpm_oracle.c for the reference file:line map.
"""
from .oracle import (IMAGE_NAMES, dpm, derive3d, layout, load, moment_indices, moments2d,
                     naive, naive_direct, num_images, project, set_threads, max_threads, synth_noise)

__all__ = ["IMAGE_NAMES", "dpm", "derive3d", "layout", "load", "moment_indices", "moments2d",
           "naive", "naive_direct", "num_images", "project", "set_threads", "max_threads", "synth_noise"]
