"""Multi-GPU: 2D block-cyclic Cholesky with panel broadcasts."""
from .cholesky_dist import B200Ops, Comm, Ops, TorchComm, cholesky_distributed
from .layout import BlockCyclic2D, grid_for

__all__ = ["BlockCyclic2D", "grid_for", "cholesky_distributed", "TorchComm", "B200Ops", "Comm", "Ops"]
