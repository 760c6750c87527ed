#!/bin/bash
# Winograd / FFT transform kernels + SGD: CUDA-event times, then the ncu launch list
# with DRAM bytes (HBM GB/s per kernel).
out=gpurun_out; mkdir -p $out; tag=${1:-r02}
timeout 300 python scripts/family_profile.py 10 > $out/${tag}_family_times.json 2> $out/${tag}_family.err && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $out/${tag}_family_launches.csv python scripts/family_profile.py 1 > $out/${tag}_family_ncu.log 2>&1
echo "rc=$?"
