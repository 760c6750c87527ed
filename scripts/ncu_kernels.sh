#!/bin/bash
# Targeted `ncu --set full` captures of the hot kernels of one ResNet-50 bs256
# bf16 training step (scripts/step_profile.py), one capture per kernel class;
# raw-page CSVs land in gpurun_out/<tag>_ncu_<name>.csv.
#   gpurun --timeout 2400 -- bash scripts/ncu_kernels.sh r01
tag=${1:-r01}
out=gpurun_out
mkdir -p $out
timeout 300 python scripts/step_profile.py > $out/${tag}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
cap() {  # name regex count skip
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    --kernel-name-base demangled -k "regex:$2" -c "$3" -s "${4:-0}" -o /tmp/${tag}_$1 -f python scripts/step_profile.py \
    > $out/${tag}_ncu_$1.log 2>&1
  ncu -i /tmp/${tag}_$1.ncu-rep --page raw --csv > $out/${tag}_ncu_$1.csv 2>> $out/${tag}_ncu_$1.log
  ncu -i /tmp/${tag}_$1.ncu-rep --page details --csv > $out/${tag}_ncu_$1_details.csv 2>> $out/${tag}_ncu_$1.log
}
cap fwd_epi "conv_tc_kernel<\\(tcb::ConvMode\\)0, \\(int\\)256, \\(int\\)1, \\(int\\)2, \\(bool\\)0>" 2
cap dgrad_epi "conv_tc_kernel<\\(tcb::ConvMode\\)1, \\(int\\)256, \\(int\\)1, \\(int\\)2, \\(bool\\)0>" 2
cap fwd_3x3_cta2 "conv_tc_kernel<\\(tcb::ConvMode\\)0, \\(int\\)256, \\(int\\)2, \\(int\\)0, \\(bool\\)1>" 2
cap dgrad_3x3_cta2 "conv_tc_kernel<\\(tcb::ConvMode\\)1, \\(int\\)128, \\(int\\)2, \\(int\\)0, \\(bool\\)1>" 2
cap wgrad_3x3_cta2 "conv_tc_kernel<\\(tcb::ConvMode\\)2, \\(int\\)256, \\(int\\)2, \\(int\\)0, \\(bool\\)1>" 2
cap wgrad_1x1_cta2 "conv_tc_kernel<\\(tcb::ConvMode\\)2, \\(int\\)256, \\(int\\)1, \\(int\\)0, \\(bool\\)1>" 2
cap dgrad_phase_staged "conv_tc_kernel<\\(tcb::ConvMode\\)1, \\(int\\)128, \\(int\\)2, \\(int\\)0, \\(bool\\)0>" 4
cap window "conv_win_kernel|conv_win_wgrad_kernel" 2
cap stem "conv_stem|maxpool" 3
cap misc "split_reduce|sgd4|dgrad_empty" 4
du -sh $out
