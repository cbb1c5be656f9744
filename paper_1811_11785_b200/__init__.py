"""B200-native SVD-PHAT / SRP-PHAT per-frame localisation (arXiv 1811.11785).

The product is libsvdphat.so (C-ABI in include/svdphat.h, CUDA kernels for sm_100a in csrc/); this package is its
thin Python binding.  Importing it loads the shared library and fails loudly if it is missing.
"""
from ._lib import (DUMP_CLASS_REP, DUMP_KEYS, DUMP_PHASORS, DUMP_POWER, DUMP_Z, LIB_PATH,  # noqa: F401
                   OPT_DAS, OPT_DAS_FOLD, OPT_NO_DAS, OPT_NO_SRP_FOLD, OPT_NO_SVD_FOLD, OPT_ONE_CTA_PROJ, OPT_ONE_CTA_SRP, Plan, SvdPhatError,
                   frame_count, lib)
