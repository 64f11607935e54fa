"""B200-native overdecomposed Jacobi3D (arxiv 2605.12734's overdecomposition hot path).

The product is the C-ABI library ``libjacobi3d.so`` (include/jacobi3d.h); this
package holds its CUDA/C++ sources (``csrc/``), the in-tree build (``build.py``),
the ctypes binding (``jacobi3d.py``) and the one-process-per-GPU plumbing over
torch.distributed (``dist.py``).  It never imports ``oracle/``.
"""
from .jacobi3d import *  # noqa: F401,F403
from .jacobi3d import Jacobi2D, Jacobi3D, JacError, load  # noqa: F401

__version__ = "0.1.0"
