"""B200-native (sm_100a) compressed clustered neighbor list — a drop-in for the
build-and-query path of arXiv 2602.19873's reference (``/root/reference/proj``).

The compute path is ``libsfcnl_b200.so`` (hand-written CUDA, C-ABI in
``include/sfcnl_cu.h``); this package is the host-side mirror of the
reference's public API over that ABI. See DESIGN.md.
"""
from .api import *  # noqa: F401,F403
from .api import (BuildError, BuildParams, ClusterParams, Context, DecodeError, EvrardSpec,  # noqa: F401
                  InputError, NeighborStore, Octree, ParticleSet, PassConfig, ReduceResult,
                  SfcOrder, SimulationBox, UniformSpec)
from .pipeline import Pipeline, StreamedPipeline  # noqa: F401
