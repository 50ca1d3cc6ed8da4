"""B200-native docking hot path of arXiv 2209.05069 (LiGen-style geometric docking).

Mirror of the reference package `dockscreen`: the same modules, names and error
behaviour, with the native slot `dockscreen.kernels._core` (pkg/setup.py:10-18) replaced by
libdockscreen.so — hand-written sm_100a CUDA kernels behind a C ABI (include/dockscreen.h).
"""
from . import model
from .model import (Atom, Counters, DockConfig, DockResult, Fragment, Ligand, Pocket, Pose, validate_ligand,
                    TooManyAtoms, MalformedFragment, IndexOutOfRange, DegenerateAxis, NoValidPose, EmptyPocket,
                    InfeasibleShape)

__all__ = ["model", "Atom", "Counters", "DockConfig", "DockResult", "Fragment", "Ligand", "Pocket", "Pose",
           "validate_ligand", "TooManyAtoms", "MalformedFragment", "IndexOutOfRange", "DegenerateAxis",
           "NoValidPose", "EmptyPocket", "InfeasibleShape"]
