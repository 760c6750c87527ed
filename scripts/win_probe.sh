#!/bin/bash
# Window conv vs im2col-TMA path on the ResNet-50 3x3 layers (bs256): times
# (CUDA events) then one ncu --set full capture of the window kernel per case.
out=gpurun_out; mkdir -p $out; tag=${1:-r02w}
cases=("256 56 56 64 64 3 3 1 1" "256 28 28 128 128 3 3 1 1" "256 14 14 256 256 3 3 1 1")
for c in "${cases[@]}"; do
  for p in fwd dgrad; do
    for w in 1 0; do
      echo "win=$w $c $p $(TCB_WIN=$w timeout 120 python scripts/conv_bench.py $c $p 20)" >> $out/${tag}_times.txt
    done
  done
done
cat $out/${tag}_times.txt
[ "${SKIP_NCU:-0}" = 1 ] && exit 0
i=0
for c in "${cases[@]:0:2}"; do
  for p in fwd dgrad; do
    timeout 300 ncu --set full --clock-control none --import-source on -k regex:conv_win_kernel -s 3 -c 1 \
      -o /tmp/${tag}_$i -f python scripts/conv_bench.py $c $p 5 > $out/${tag}_ncu_$i.log 2>&1
    ncu -i /tmp/${tag}_$i.ncu-rep --page raw --csv > $out/${tag}_ncu_$i.csv 2>> $out/${tag}_ncu_$i.log
    ncu -i /tmp/${tag}_$i.ncu-rep --page source --csv > $out/${tag}_ncu_${i}_src.csv 2>> $out/${tag}_ncu_$i.log
    ncu -i /tmp/${tag}_$i.ncu-rep --page details --csv > $out/${tag}_ncu_${i}_details.csv 2>> $out/${tag}_ncu_$i.log
    i=$((i+1))
  done
done
