# A/B of TCB_CTA2_KB (CTA pairs for layers with at least this many k-blocks), whole steps
set -u
mkdir -p gpurun_out; : > gpurun_out/abcta2.txt
run() { m=$1; b=$2; v=$3; f=gpurun_out/abcta2_${m}_${v}.json
  TCB_CTA2_KB=$v timeout 300 python bench.py --model $m --batch $b --steps 20 --warmup 4 --no-cpu-baseline --no-roofline --no-e2e 2>/dev/null | tail -1 > $f
  python -c "import json;d=json.load(open('$f'));print('$m','$v',d['value'],d['ms_per_step'])" >> gpurun_out/abcta2.txt 2>&1; }
for m in "resnet50 256" "inception_v3 128" "vgg16 64"; do
  set -- $m
  for v in 9 4 6 12 16 24 9; do run $1 $2 $v; done
done
cat gpurun_out/abcta2.txt
