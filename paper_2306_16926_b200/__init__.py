"""B200-native OSP synchronization hot path (arXiv 2306.16926).

split -> RS push/aggregate/pull -> LGP -> ICS push/aggregate/correct -> PGP ->
next GIB, as hand-written sm_100a kernels behind a C-ABI (include/osp_c.h),
with the reference pslab worker/server semantics. See DESIGN.md.
"""
import importlib

from . import layouts
from ._capi import LIB_PATH, load

__all__ = ["layouts", "load", "LIB_PATH"]


def __getattr__(name):
    # torch-backed front, imported lazily so the C-ABI can be probed without it
    if name.startswith("__"):
        raise AttributeError(name)
    osp = importlib.import_module(__name__ + ".osp")
    if name == "osp":
        return osp
    if hasattr(osp, name):
        return getattr(osp, name)
    raise AttributeError(name)
