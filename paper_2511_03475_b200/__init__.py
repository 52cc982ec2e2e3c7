"""B200-native RAGBoost context index (arXiv 2511.03475): CUDA kernels for
sm_100a behind the C-ABI in include/ragb.h, and this thin binding."""
from .ragb import (RB_ALPHA_ANY, RB_EMIT_COUNTS, RB_KEEP_ROWS, RB_SKIP_LINKAGE, Index, RagbError,  # noqa: F401
                   Session, Workspace, build_index, build_index_host, index_from_linkage, version,
                   workspace_size, make_params)
