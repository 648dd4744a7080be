set -u
O=gpurun_out/r02q2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/_mut_lag1_tmp.py -q -k "dedicated" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
