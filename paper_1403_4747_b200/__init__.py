"""B200-native fast directional algorithm (FDA) for the Burton-Miller BEM.

Cao, Wen & Xiao, "A fast directional boundary element method for high
frequency acoustic problems in three dimensions" (arXiv 1403.4747).
The product is libfda.so (include/fda.h); ``fda.FDA`` is its Python binding.
"""
from .fda import FDA, FdaError, load_library, default_options, exchange_local, EXPORTS, STAGES  # noqa: F401
