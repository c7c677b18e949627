"""B200-native mQO inner loop (arXiv 2605.06921): CUDA kernels for sm_100a
behind the C ABI of include/mqo_gpu.h, with a Python mirror of the
reference's C++ API.  Importing this package loads libmqo_b200.so and fails
loudly if it is missing -- there is no CPU fallback."""
from . import _lib  # noqa: F401  (loads the shared library)
from .api import *  # noqa: F401,F403
from .api import __all__ as _api_all

__all__ = list(_api_all)
__version__ = _lib.lib.mqo_version().decode()
