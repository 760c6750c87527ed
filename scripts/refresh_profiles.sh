#!/bin/bash
# Round-end evidence refresh (one GPU): in-step conv table, launch list with
# DRAM bytes (roofline.traffic), ncu --set full per kernel class.
#   gpurun --timeout 3000 -- bash scripts/refresh_profiles.sh <tag>
tag=${1:-r01}
out=gpurun_out
mkdir -p $out
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $out/${tag}_bench.json 2> $out/${tag}_bench.err || exit 1
cp $out/conv_in_step_resnet50_bf16.json $out/${tag}_conv_in_step.json
timeout 600 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none --csv --log-file $out/${tag}_traffic.csv python scripts/step_profile.py > $out/${tag}_traffic.log 2>&1
bash scripts/ncu_kernels.sh $tag
