"""paper_2305_06942_b200 -- B200-native fused EmbeddingBag(sum) + All-to-All.

The data-parallel hot path of arXiv 2305.06942 (Sec 3.2-3.3): each GPU sum-pools its
model-parallel tables for the whole global batch and stores every pooled vector zero-copy into
the destination GPU's data-parallel receive buffer over NVLink, signalling per-peer arrival
counters with system-scope release/acquire, inside one sm_100a kernel.

Public API: EmbA2A (one rank), LoopbackGroup (W virtual ranks on one device), LocalGroup /
torch_allgather (bootstrap channels).  C ABI: include/emb_a2a.h, libemba2a.so.
Row f4: AgGemm / AgGemmLoopback, the fused AllGather + GEMM (include/ag_gemm.h).
"""
from ._lib import LIB_PATH, EXPORTED  # noqa: F401  (raises if the library is not built)
from .emb_a2a import (EmbA2A, EmbA2AError, LocalGroup, run_ranks,  # noqa: F401
                      torch_allgather)
from .loopback import LoopbackGroup  # noqa: F401
from .ag_gemm import AgGemm, AgGemmLoopback  # noqa: F401
