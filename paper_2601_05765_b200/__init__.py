"""B200-native (sm_100a) partial-optimal-transport hot path of arXiv 2601.05765.

Package layout mirrors the reference ``potflow`` entry points for the hot
path (/root/reference/pkg/src/potflow/__init__.py:10-20):

geom        host geometry: planes, convex cells, domain pack     (geom.py)
laguerre    device bucket grid, kNN, weight reductions           (laguerre.py)
_kernels    drop-in for the reference batch kernels              (_kernels.py)
restricted  torch-level evaluation of restricted Laguerre cells  (SPEC restricted_cell)
solver      damped Newton (KMT) solve for the weights            (SPEC ot_solver)
fluid       advection + barycentric spring step                  (SPEC fluid_sim)

All per-cell work runs in libpotflow_b200.so (hand-written CUDA for sm_100a,
loaded through ctypes).  There is no CPU fallback.
"""
__version__ = "0.1.0"


def set_threads(n: int) -> int:
    """Reference API (__init__.py:33-44).  Device kernels have no host thread
    count; results are independent of it, as in the reference."""
    return max(1, int(n))


def set_parity_mode(on: bool) -> None:
    """Reference-faithful restriction on every evaluation of this device
    (DESIGN.md §5.1); default off (the robust restriction)."""
    from ._lib import set_parity_mode as _s

    _s(on)


def library_path() -> str:
    from ._lib import LIB_PATH

    return LIB_PATH
