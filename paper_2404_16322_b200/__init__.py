"""B200-native DADE hot path (arxiv 2404.16322): C-ABI library libdade.so + thin binding."""
from .dade import Index, DadeError, Stats, lib, LIB_PATH, MAX_K, MAX_STEPS  # noqa: F401
