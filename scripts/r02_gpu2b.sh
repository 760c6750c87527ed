#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_ps_multigpu.py -m gpu -q -p no:cacheprovider > $out/r02h_ps.log 2>&1; echo "ps rc=$?" >> $out/r02h_ps.log; tail -3 $out/r02h_ps.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-cpu-baseline > $out/r02h_bench_g1.json 2> $out/r02h_bench_g1.err; echo "g1 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 > $out/r02h_bench_g2.json 2> $out/r02h_bench_g2.err; echo "g2 rc=$?"
