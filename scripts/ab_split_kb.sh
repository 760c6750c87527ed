# A/B of TCB_SPLIT_MIN_KB (wgrad split-K: fewest k-blocks per split), whole steps on C3/C4/C5
set -u
mkdir -p gpurun_out; : > gpurun_out/absplit.txt
run() { m=$1; b=$2; v=$3; f=gpurun_out/absplit_${m}_${v}.json
  TCB_SPLIT_MIN_KB=$v timeout 300 python bench.py --model $m --batch $b --steps 20 --warmup 4 --no-cpu-baseline --no-roofline --no-e2e 2>/dev/null | tail -1 > $f
  python -c "import json;d=json.load(open('$f'));print('$m','$v',d['value'],d['ms_per_step'])" >> gpurun_out/absplit.txt 2>&1; }
for m in "resnet50 256" "inception_v3 128" "vgg16 64"; do
  set -- $m
  for v in 4 2 8 16 32 4; do run $1 $2 $v; done
done
cat gpurun_out/absplit.txt
