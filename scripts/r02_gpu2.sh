#!/bin/bash
# 2-GPU evidence pass: measured tf32/ffma peaks, NVLink peak + counters, NVLS/NCCL
# PS microbenchmark with NVLink byte counters, 1- and 2-GPU bench lines.
out=gpurun_out; mkdir -p $out
timeout 300 python scripts/measure_peaks.py > $out/r02_measured_peaks_tf32_ffma.json 2> $out/r02_peaks.err
timeout 300 python scripts/nvlink_peak.py > $out/r02_nvlink_peak_g2.json 2> $out/r02_nvlink_peak.err
timeout 600 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 scripts/nvls_bench.py > $out/r02_nvls_bench_g2.json 2> $out/r02_nvls_bench_g2.err
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > $out/r02_bench_g1.json 2> $out/r02_bench_g1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 > $out/r02_bench_g2.json 2> $out/r02_bench_g2.err
ls -la $out | tail -20
