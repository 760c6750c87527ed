# A/B of TCB_EPI_DEEP_KB (whole-share side-input prefetch in the TMA epilogue), whole steps
set -u
mkdir -p gpurun_out; : > gpurun_out/abdeep.txt
run() { m=$1; b=$2; v=$3; f=gpurun_out/abdeep_${m}_${v}.json
  TCB_EPI_DEEP_KB=$v timeout 300 python bench.py --model $m --batch $b --steps 20 --warmup 4 --no-cpu-baseline --no-roofline --no-e2e 2>/dev/null | tail -1 > $f
  python -c "import json;d=json.load(open('$f'));print('$m','$v',d['value'],d['ms_per_step'])" >> gpurun_out/abdeep.txt 2>&1; }
for m in "resnet50 256" "vgg16 64" "inception_v3 128"; do
  set -- $m
  for v in 2 0 4 8 12 2; do run $1 $2 $v; done
done
cat gpurun_out/abdeep.txt
