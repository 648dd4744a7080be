#!/bin/bash
# Round-2 evidence in one GPU call: tests, sanitizers, smoke (+ its ncu launch list), the default
# bench line, the reference arm, the AllGather+GEMM line, the bench matrix, DRAM traffic of every
# config (profiles/ncu_traffic.json), a launch list of the default bench command, and one
# `ncu --set full` capture each of the fused forward and the AllGather+GEMM kernel.
set -u
tag=${1:-r02y}
O=gpurun_out/$tag; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_smoke.py > $O/san_$t.log 2>&1; echo "rc=$?" >> $O/san_$t.log
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_smoke.py --W 2 > $O/san_memcheck_W2.log 2>&1; echo "rc=$?" >> $O/san_memcheck_W2.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_ncu.log 2>&1; echo "rc=$?" >> $O/smoke_ncu.log
bash tools/ncu_traffic.sh $tag > $O/ncu_traffic.log 2>&1
python tools/ncu_traffic.py gpurun_out/ncu_$tag $O/ncu_traffic.json > /dev/null 2>&1
cp $O/ncu_traffic.json profiles/ncu_traffic.json
timeout 900 python bench.py --out $O/bench.jsonl > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
timeout 900 python bench.py --impl reference > $O/bench_reference.log 2>&1; echo "rc=$?" >> $O/bench_reference.log
timeout 900 python bench.py --path ag_gemm --out $O/ag.jsonl > $O/ag.log 2>&1; echo "rc=$?" >> $O/ag.log
timeout 900 python bench.py --path ag_gemm --ag-config ag_small --no-cpu --steps 50 --out $O/ag.jsonl > $O/ag_small.log 2>&1
timeout 900 python bench.py --path ag_gemm --impl reference --steps 2 --warmup 1 > $O/ag_reference.log 2>&1
bash tools/bench_matrix.sh $tag > $O/matrix.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv python bench.py --steps 10 --warmup 3 --no-cpu --ag-leg 0 > $O/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:emb_a2a_kernel -s 12 -c 1 -o $O/fwd_full python bench.py --steps 10 --warmup 3 --no-cpu --no-baseline --no-backward --no-alpha0 --ag-leg 0 > $O/ncu_fwd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ag_gemm_kernel -s 3 -c 1 -o $O/ag_full python bench.py --path ag_gemm --steps 3 --warmup 2 --no-cpu > $O/ncu_ag.log 2>&1
echo done > $O/DONE
