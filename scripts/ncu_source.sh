#!/bin/bash
# One `ncu --set full --import-source on` capture of a single kernel class of the
# step, exported as the source (SASS) page with per-instruction stall samples.
#   gpurun -- bash scripts/ncu_source.sh <tag> <regex> [skip]
tag=$1; rx=$2; skip=${3:-0}
out=gpurun_out; mkdir -p $out
timeout 300 python scripts/step_profile.py > $out/${tag}_plain.log 2>&1 || exit 1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  --kernel-name-base demangled -k "regex:$rx" -c 1 -s $skip -o /tmp/${tag} -f python scripts/step_profile.py \
  > $out/${tag}_ncu.log 2>&1
ncu -i /tmp/${tag}.ncu-rep --page source --csv --print-source sass > $out/${tag}_source.csv 2>> $out/${tag}_ncu.log
ncu -i /tmp/${tag}.ncu-rep --page details --csv > $out/${tag}_details.csv 2>> $out/${tag}_ncu.log
ncu -i /tmp/${tag}.ncu-rep --page raw --csv > $out/${tag}_raw.csv 2>> $out/${tag}_ncu.log
