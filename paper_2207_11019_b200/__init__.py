"""pipeplan_b200: B200-native layer-wise partition-and-merge training step.

Host-side mirror of the reference `pipeplan` API for the hot path
(`train_partitioned` and the planner it consumes), backed by the C ABI in
include/pipeplan_b200.h and hand-written sm_100a kernels (libpipeplan_b200.so,
built in-tree).  Importing does not load the library; the first call does, and
raises if it is missing.
"""
from .api import *  # noqa: F401,F403
from .api import __all__  # noqa: F401
