#!/bin/bash
# 2/4-GPU pass: weak-scaling bench (with e2e; PS step over NVSwitch multicast by
# default, NCCL for A/B), NCCL busbw + NVLS microbench, VGG-16 N_ps sweep,
# multi-GPU PS tests.
#   gpurun --gpus 4 --timeout 2400 -- bash scripts/multi_gpu_check.sh <tag>
tag=${1:-r01}
out=gpurun_out
mkdir -p $out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python bench.py --no-cpu-baseline > $out/${tag}_bench_g1.json 2> $out/${tag}_bench_g1.err
timeout 600 $TR --nproc-per-node 2 --master-port 29511 bench.py --gpus 2 --no-cpu-baseline > $out/${tag}_bench_g2.json 2> $out/${tag}_bench_g2.err
timeout 600 $TR --nproc-per-node 4 --master-port 29512 bench.py --gpus 4 --no-cpu-baseline > $out/${tag}_bench_g4.json 2> $out/${tag}_bench_g4.err
timeout 600 $TR --nproc-per-node 4 --master-port 29513 bench.py --gpus 4 --no-cpu-baseline --ps-transport nccl > $out/${tag}_bench_g4_nccl.json 2> $out/${tag}_bench_g4_nccl.err
timeout 300 $TR --nproc-per-node 4 --master-port 29515 scripts/nvls_bench.py > $out/${tag}_nvls_bench_g4.json 2> $out/${tag}_nvls_bench_g4.err
timeout 300 $TR --nproc-per-node 4 --master-port 29514 scripts/nccl_busbw.py > $out/${tag}_busbw_g4.json 2> $out/${tag}_busbw_g4.err
for n in 1 2 4; do
  timeout 600 $TR --nproc-per-node 4 --master-port 2952$n bench.py --gpus 4 --model vgg16 --batch 64 --n-ps $n --no-cpu-baseline --no-e2e \
    > $out/${tag}_vgg_g4_nps$n.json 2> $out/${tag}_vgg_g4_nps$n.err
done
timeout 600 $TR --nproc-per-node 4 --master-port 29529 bench.py --gpus 4 --model vgg16 --batch 64 --n-ps 4 --ps-transport nccl --no-cpu-baseline --no-e2e \
  > $out/${tag}_vgg_g4_nps4_nccl.json 2> $out/${tag}_vgg_g4_nps4_nccl.err
timeout 900 python -m pytest tests/test_ps_multigpu.py -x -q -p no:cacheprovider --timeout 300 > $out/${tag}_pytest_multigpu.log 2>&1
echo "rc=$?" >> $out/${tag}_pytest_multigpu.log
