#!/bin/bash
# Bench every BASELINE.json config (per-rank work at W=1 on one GPU) and the f2 variants.
# Output: gpurun_out/matrix_<tag>.jsonl (one bench JSON line per run).
tag=${1:-r02}
out=gpurun_out/matrix_$tag.jsonl
mkdir -p gpurun_out
run() { timeout 900 python bench.py --no-cpu --ag-leg 0 --steps 30 --alpha0-batches 2 "$@" 2>>gpurun_out/matrix_$tag.err | tail -1 >> $out; echo "done: $*"; }
run --config dlrm_small
run --config dlrm_small --table-dtype bf16
run --config dlrm_small --table-dtype f16
run --config dlrm_small --out-dtype bf16
run --config dlrm_small --pooling mean
run --config dlrm_small --weighted
run --config weak
run --config sweep_p1 --batches 8
run --config sweep_p4 --batches 8
run --config sweep_p8 --batches 8
run --config sweep_p32 --batches 4
run --config sweep_p128 --batches 2 --steps 20 --no-alpha0
run --config dlrm_wide --batches 4
run --config dlrm_wide --batches 4 --table-dtype bf16
run --config dlrm_wide --batches 4 --out-dtype bf16
