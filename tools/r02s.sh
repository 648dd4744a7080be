set -u
O=gpurun_out/r02s; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
run() { timeout 600 python bench.py --no-cpu --no-alpha0 --no-backward --no-baseline --ag-leg 0 --steps 30 "$@" 2>>$O/err.log | tail -1 >> $O/chunk.jsonl; }
for c in 16 32 64 128 256; do run --config sweep_p1 --batches 8 --chunk $c; done
for c in 16 32 64 128; do run --config sweep_p4 --batches 8 --chunk $c; done
for c in 16 32 64; do run --config dlrm_small --chunk $c; done
for c in 16 32 64; do run --config weak --chunk $c; done
