#!/bin/bash
# One GPU-box pass: tests, smoke, default bench (both arms), then ncu captures
# of the hot kernels of one training step (only after the plain run exited 0).
#   gpurun --timeout 3000 -- bash scripts/gpu_check.sh [tag]
tag=${1:-r01}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $out/${tag}_gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $out/${tag}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $out/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/${tag}_smoke.log 2>&1
echo "smoke rc=$?" >> $out/${tag}_smoke.log
timeout 600 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err
rc=$?
echo "bench rc=$rc" >> $out/${tag}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/${tag}_bench_ref.json 2> $out/${tag}_bench_ref.err
echo "ref rc=$?" >> $out/${tag}_bench_ref.err
if [ $rc -eq 0 ] && [ "${SKIP_NCU:-0}" != 1 ]; then
  timeout 300 python scripts/step_profile.py > $out/${tag}_step_plain.log 2>&1 && \
  timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"${NCU_KERNELS:-conv_tc|sgd|split_reduce|maxpool|im2col}" -c ${NCU_COUNT:-16} \
    -o /tmp/${tag}_full -f python scripts/step_profile.py > $out/${tag}_ncu_full.log 2>&1
  echo "ncu rc=$?" >> $out/${tag}_ncu_full.log
  ncu -i /tmp/${tag}_full.ncu-rep --page raw --csv > $out/${tag}_ncu_raw.csv 2>> $out/${tag}_ncu_full.log
  ncu -i /tmp/${tag}_full.ncu-rep --page details --csv > $out/${tag}_ncu_details.csv 2>> $out/${tag}_ncu_full.log
  sz=$(stat -c %s /tmp/${tag}_full.ncu-rep 2>/dev/null || echo 0)
  [ "$sz" -lt 30000000 ] && cp /tmp/${tag}_full.ncu-rep $out/
fi
du -sh $out
