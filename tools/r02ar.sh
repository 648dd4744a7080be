#!/bin/bash
# r02ar: the SCALE command shape at N = 4 and 8 with the default config, all ranks sharing the
# one GPU (EMBA2A_SHARED_GPU=1): bootstrap, cudaIpc mapping, parity, the JSON line (timings are
# meaningless with shared SMs)
set -u
O=gpurun_out/${1:-r02ar}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for n in 4 8; do
  EMBA2A_SHARED_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29500 + n)) bench.py --gpus $n --steps 5 --warmup 3 \
    > $O/n$n.out 2> $O/n$n.err
  echo "n=$n rc=$?" >> $O/rc.txt
done
