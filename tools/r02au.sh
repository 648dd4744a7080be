set -u
O=gpurun_out/r02au; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
run() { timeout 300 python bench.py --no-cpu --no-alpha0 --no-baseline --ag-leg 0 --steps 30 "$@" 2>>$O/err.log | tail -1 >> $O/bwd.jsonl; }
for c in dlrm_small weak sweep_p1; do
  for cap in 8192 4096 2048; do run --config $c --opt sort_mode=5 --opt bucket_cap=$cap; done
done
