#!/bin/bash
# NVSwitch-multicast PS step: 2-GPU parity tests, then bench.py both transports.
#   gpurun --gpus 2 --timeout 1500 -- bash scripts/nvls_check.sh [G]
G=${1:-2}
out=gpurun_out
mkdir -p $out
timeout 600 python -m pytest tests/test_ps_multigpu.py -q -x -p no:cacheprovider > $out/nvls_pytest.log 2>&1
echo "pytest rc=$?" >> $out/nvls_pytest.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1"
for tp in nccl nvls; do
  timeout 400 $TR --master-port 2960$G bench.py --gpus $G --steps 20 --warmup 5 --ps-transport $tp --no-cpu-baseline \
    > $out/nvls_bench_g${G}_$tp.json 2> $out/nvls_bench_g${G}_$tp.err
  echo "rc=$?" >> $out/nvls_bench_g${G}_$tp.err
done
