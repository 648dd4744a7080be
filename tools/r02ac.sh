set -u
O=gpurun_out/r02ac; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
run() { timeout 600 python bench.py --no-cpu --no-alpha0 --no-backward --no-baseline --ag-leg 0 --steps 40 "$@" 2>>$O/err.log | tail -1 >> $O/sweep.jsonl; }
for c in dlrm_small weak; do
  run --config $c
  for v in 2 4; do run --config $c --opt vec=$v; done
  for t in 128 192; do run --config $c --opt threads=$t; done
  for st in 2 3 6; do run --config $c --opt stages=$st; done
  for fb in 0 32; do run --config $c --opt flat_below=$fb; done
  run --config $c --opt ctas_per_sm=3
  run --config $c
done
