set -u
O=gpurun_out/r02u; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_protocol.py tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
run() { timeout 600 python bench.py --no-cpu --no-alpha0 --no-backward --no-baseline --ag-leg 0 --steps 30 "$@" 2>>$O/err.log | tail -1 >> $O/chunk.jsonl; }
for c in 32 48 64 96 127; do run --config sweep_p1 --batches 8 --chunk $c; done
for c in 32 64 127; do run --config sweep_p4 --batches 8 --chunk $c; done
for c in 32 48 64; do run --config sweep_p8 --batches 8 --chunk $c; done
for c in 32 48 64; do run --config dlrm_small --chunk $c; done
for c in 32 48 64; do run --config weak --chunk $c; done
for c in 32 64; do run --config dlrm_wide --batches 4 --chunk $c; done
