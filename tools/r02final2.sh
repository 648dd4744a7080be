#!/bin/bash
# Final-build evidence without the sanitizers (closed on the pool) and the ncu traffic captures
# (kernels unchanged since r02ao): tests, smoke (+ ncu launch list), default bench line, the
# reference arm, the AllGather+GEMM lines, the bench matrix, the default bench's launch list.
set -u
tag=${1:-r02az}
O=gpurun_out/$tag; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_ncu.log 2>&1; echo "rc=$?" >> $O/smoke_ncu.log
timeout 900 python bench.py --out $O/bench.jsonl > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
timeout 900 python bench.py --impl reference > $O/bench_reference.log 2>&1; echo "rc=$?" >> $O/bench_reference.log
timeout 900 python bench.py --path ag_gemm --out $O/ag.jsonl > $O/ag.log 2>&1; echo "rc=$?" >> $O/ag.log
bash tools/bench_matrix.sh $tag > $O/matrix.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv python bench.py --steps 10 --warmup 3 --no-cpu --ag-leg 0 > $O/launches_bench.log 2>&1
echo done > $O/DONE
