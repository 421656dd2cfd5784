"""paper_2511_02062_b200 — B200-native retrieval stage of Vortex (arXiv 2511.02062).

Exact inner-product top-k over a sharded embedding index + ColBERT/PreFLMR MaxSim
re-scoring, behind the reference's operator API (ComponentFn; see component.py and
include/vortex_b200_component.hpp).  Compute is hand-written sm_100a CUDA in
csrc/, reached through the C-ABI of include/vortex_b200.h (libvortex_b200.so).
"""
from ._lib import (VX_COARSE_AUTO, VX_COARSE_BF16, VX_COARSE_I8, VX_COARSE_TF32,
                   VX_FLAG_NO_BF16_SHADOW, VX_FLAG_NO_I8_SHADOW, VX_FLAG_TOKENS_F32,
                   VX_MAXSIM_AUTO, VX_MAXSIM_CC, VX_MAXSIM_TC, VX_MAXSIM_TC_BF16Q, VX_OPT_COARSE, VX_OPT_GRAPHS,
                   VX_OPT_GRID, VX_OPT_KPRIME, VX_OPT_MAXSIM, VX_OPT_SCAN, VX_OPT_SCAN_PAIRS,
                   VX_OPT_SCAN_SEED, VX_OPT_SCAN_TILE, VX_OPT_I8_SCALE, VX_OPT_STAGE_EVENTS,
                   VX_PREPARE_RESCORE, VX_PREPARE_SEARCH, VX_SCAN_AUTO,
                   VX_SCAN_F32, VX_SCAN_TC, VxError, load)
from .component import (Registry, SearchComponent, VortexError, decode_query, decode_result,
                        encode_query, encode_result)
from .index import Index

__all__ = ["Index", "SearchComponent", "Registry", "VortexError", "VxError", "load",
           "encode_query", "decode_query", "encode_result", "decode_result", "VX_SCAN_AUTO",
           "VX_SCAN_F32", "VX_SCAN_TC", "VX_OPT_SCAN", "VX_OPT_GRID", "VX_OPT_GRAPHS", "VX_OPT_MAXSIM",
           "VX_MAXSIM_AUTO", "VX_MAXSIM_CC", "VX_MAXSIM_TC", "VX_MAXSIM_TC_BF16Q", "VX_PREPARE_SEARCH", "VX_PREPARE_RESCORE"]
