#!/bin/bash
# TF32 tensor-core mode evidence: launch list of one ResNet-50 bs256 tf32 step
# plus one `ncu --set full` capture of representative conv_tf32 launches.
#   gpurun --timeout 1500 -- bash scripts/tf32_ncu.sh
out=gpurun_out
mkdir -p $out
timeout 300 python scripts/step_profile.py resnet50 256 tf32 > $out/tf32_step_plain.log 2>&1 || exit 1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_op_tmem_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none --csv --log-file $out/tf32_launches.csv python scripts/step_profile.py resnet50 256 tf32 > $out/tf32_ncu_launch.log 2>&1
echo "launch rc=$?" >> $out/tf32_ncu_launch.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:conv_tf32 -c 6 -o /tmp/tf32_full -f python scripts/step_profile.py resnet50 256 tf32 > $out/tf32_ncu_full.log 2>&1
echo "full rc=$?" >> $out/tf32_ncu_full.log
ncu -i /tmp/tf32_full.ncu-rep --page raw --csv > $out/tf32_ncu_raw.csv 2>> $out/tf32_ncu_full.log
