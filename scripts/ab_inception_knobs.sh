set -u
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --model inception_v3 --batch 128 --steps 15 --warmup 4 --no-cpu-baseline --no-roofline --no-e2e 2>/dev/null | tail -1 > gpurun_out/abinc_$tag.json; python -c "import json;d=json.load(open('gpurun_out/abinc_$tag.json'));print('$tag',d['value'],d['ms_per_step'])" >> gpurun_out/abinc.txt 2>&1; }
run base X=1
run cta2off TCB_CTA2=0
run cta2kb5 TCB_CTA2_KB=5
run cta2kb13 TCB_CTA2_KB=13
run epi4 TCB_CONV_EPI_KB=4
run epi16 TCB_CONV_EPI_KB=16
run deep0 TCB_EPI_DEEP_KB=0
run deep4 TCB_EPI_DEEP_KB=4
run base2 X=1
cat gpurun_out/abinc.txt
