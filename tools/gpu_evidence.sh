#!/bin/bash
# One GPU call's worth of evidence for profiles/: bench line, ncu launch list of the same bench
# command (cold-cache, serialised), and one `ncu --set full` capture of the fused kernel.
# Usage (on the GPU box, repo root): bash tools/gpu_evidence.sh <tag> [bench args...]
set -u
tag=${1:-r01}; shift || true
out=gpurun_out/evidence_$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > $out/gpu.csv 2>&1
timeout 900 python bench.py "$@" > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
tail -1 $out/bench.json | cut -c1-400
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/launches.csv python bench.py --steps 10 --warmup 3 --no-cpu "$@" > $out/ncu_launches.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:emb_a2a_kernel \
  -s 12 -c 1 -o $out/fused_full python bench.py --steps 10 --warmup 3 --no-cpu --no-baseline "$@" \
  > $out/ncu_full.log 2>&1
echo "ncu full rc=$?"
