"""hetbridge — B200-native boundary communicator (arxiv 2605.27678's encoder→LLM bridge).

Drop-in for the reference's ``hetsim::grid`` / ``hetsim::bridge`` surface:
layout descriptors, placement, plan compilation, and forward/backward
boundary transforms executed by hand-written sm_100a kernels over NVSwitch.
"""
from . import bridge, grid  # noqa: F401
from ._lib import HetBridgeError  # noqa: F401

__all__ = ["grid", "bridge", "autograd", "HetBridgeError"]


def __getattr__(name):  # the autograd binding imports torch; load it on first use
    if name == "autograd":
        import importlib

        return importlib.import_module(__name__ + ".autograd")
    raise AttributeError(name)
