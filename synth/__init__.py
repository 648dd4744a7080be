"""Seeded synthetic inputs for the fused EmbeddingBag + All-to-All.

This package holds NONE of the method's arithmetic: no pooling, no placement, no slicing.
It only draws the inputs both sides consume -- per-table CSR bags (Zipf-distributed row
indices, variable pooling factors) and procedural table values -- so that the CPU oracle
(oracle/) and the CUDA path (paper_2305_06942_b200/) can be fed identical data.

The paper uses "the data generator in DLRM" with no stated distribution (PAPER.md P:250,
Sec 4.1); the recipe here is the reading in DESIGN.md (R#20..R#24).
"""
from .dlrm_gen import (  # noqa: F401
    CONFIGS,
    BASE_SEED,
    ProblemConfig,
    even_partition,
    config_for,
    gen_rank_csr,
    gen_all_csr,
    table_values_host,
    splitmix64_np,
    zipf_cdf,
    to_bf16_bits,
    to_f16_bits,
    gen_weights,
)
