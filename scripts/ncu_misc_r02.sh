#!/bin/bash
# ncu --set full of the round-2 kernels outside conv_tc_kernel in one ResNet-50 bs256 bf16 step:
# sgd4 (momentum SGD), the window weight gradient, the stem weight gradient.
#   gpurun --timeout 1200 -- bash scripts/ncu_misc_r02.sh
out=gpurun_out
timeout 300 python scripts/step_profile.py > $out/r02_misc_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k "regex:sgd4_kernel|conv_win_wgrad_kernel|conv_stem_wgrad_kernel|dgrad_empty_phase" -c 4 -o /tmp/r02_misc2 -f \
  python scripts/step_profile.py > $out/r02_ncu_misc2.log 2>&1
ncu -i /tmp/r02_misc2.ncu-rep --page raw --csv > $out/r02_ncu_misc2.csv 2>> $out/r02_ncu_misc2.log
