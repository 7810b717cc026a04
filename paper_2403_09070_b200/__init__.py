"""B200-native global-placement inner loop of arXiv 2403.09070 (F2F 3D placer).

Drop-in for the ``place3d`` GP loop: ``wirelength``, ``density`` and ``gp``
keep the reference's operator names and argument meaning; every operator runs
hand-written sm_100a CUDA in ``libp3d.so`` (C-ABI: ``include/p3d.h``).  There
is no CPU fallback: importing an operator without the built library or a CUDA
device raises.
"""

from .model import (ArrayDesign, DieSpec, HbtSpec, NetlistArrays, PlacementState,
                    partition_from_z, rotate_offsets, rotated_dims)
from .synth import CONFIGS, SynthSpec, cached_synth, synth_arrays

__version__ = "0.1.0"


def __getattr__(name):
    # operator modules load libp3d.so lazily so CPU-only tooling can import the package
    if name in ("wirelength", "density", "gp", "_lib"):
        import importlib

        return importlib.import_module(f".{name}", __name__)
    if name in ("GpConfig", "GpInfo", "run_gp3d", "Gp3dProblem", "choose_grid", "init_state",
                "make_fillers", "select_flow"):
        from . import gp

        return getattr(gp, name)
    raise AttributeError(name)
