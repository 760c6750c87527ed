# A/B of TCB_CONV_EPI_KB (TMA-store epilogue up to this many k-blocks) across C3/C4/C5
set -u
mkdir -p gpurun_out; : > gpurun_out/abepi.txt
run() { m=$1; b=$2; kb=$3; f=gpurun_out/abepi_${m}_${kb}.json
  TCB_CONV_EPI_KB=$kb timeout 300 python bench.py --model $m --batch $b --steps 15 --warmup 4 --no-cpu-baseline --no-roofline --no-e2e 2>/dev/null | tail -1 > $f
  python -c "import json;d=json.load(open('$f'));print('$m','$kb',d['value'],d['ms_per_step'])" >> gpurun_out/abepi.txt 2>&1; }
for kb in 8 12 16 24 36 8; do run resnet50 256 $kb; done
for kb in 8 12 16 24 36 8; do run inception_v3 128 $kb; done
for kb in 8 16 36 8; do run vgg16 64 $kb; done
cat gpurun_out/abepi.txt
