set -u
O=gpurun_out/r02k3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $O/smi0.csv
timeout 600 python tools/ag_probe.py ag_ffn ab > $O/ab_ffn.log 2>&1
timeout 600 python tools/ag_probe.py ag_small ab > $O/ab_small.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ag_gemm.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
