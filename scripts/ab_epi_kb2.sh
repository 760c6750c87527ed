# A/B of the split 1x1 / spatial TMA-epilogue thresholds (defaults 12 / 24) vs the old single 8
set -u
mkdir -p gpurun_out; : > gpurun_out/abepi2.txt
run() { m=$1; b=$2; tag=$3; shift 3; f=gpurun_out/abepi2_${m}_${tag}.json
  env "$@" timeout 300 python bench.py --model $m --batch $b --steps 20 --warmup 4 --no-cpu-baseline --no-roofline --no-e2e 2>/dev/null | tail -1 > $f
  python -c "import json;d=json.load(open('$f'));print('$m','$tag',d['value'],d['ms_per_step'])" >> gpurun_out/abepi2.txt 2>&1; }
for m in "resnet50 256" "inception_v3 128" "vgg16 64"; do
  set -- $m
  run $1 $2 new X=1; run $1 $2 old8 TCB_CONV_EPI_KB=8; run $1 $2 s12 TCB_CONV_EPI_KB_SPATIAL=12; run $1 $2 s36 TCB_CONV_EPI_KB_SPATIAL=36; run $1 $2 new2 X=1; run $1 $2 old8b TCB_CONV_EPI_KB=8
done
cat gpurun_out/abepi2.txt
