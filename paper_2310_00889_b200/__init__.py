"""B200-native slender-body Nystrom operator apply (arXiv 2310.00889).

The product is libslb.so (hand-written CUDA for sm_100a + NCCL, C-ABI in include/slb.h);
this package is its thin ctypes binding (api) plus the rank partition helper (shard).
"""
from .api import (slb_abi_version, slb_eta_cfie, slb_coincident_count, slb_coincident_reset, slb_launch_count,
                  slb_upsample, slb_upsample_ragged, slb_farfield_laplace_dl, slb_farfield_stokes_sldl, slb_nearcorr_apply,
                  slb_nearcorr_fold, slb_fill_blocks, slb_near_build, slb_nearcorr_quad, slb_bench_dfma, Comm, Operator, LAPLACE_DL, STOKES_SLDL, STOKES_SL)
from .shard import partition_panels
from ._native import SlbError, SO_PATH
