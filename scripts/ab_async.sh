#!/bin/bash
# A/B of the asynchronous PS policy at 4 GPUs (ResNet-50 bs256, VGG-16 bs64).
#   gpurun --gpus 4 --timeout 1800 -- bash scripts/ab_async.sh
out=gpurun_out
mkdir -p $out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
: > $out/ab_async.txt
for m in "resnet50 256" "vgg16 64"; do
  set -- $m
  for mode in "" "--ps-async"; do
    timeout 400 $TR --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --model $1 --batch $2 --no-cpu-baseline --no-e2e $mode \
      > $out/ab_async_$1${mode}.json 2>/dev/null
    python -c "
import json; b=json.loads(open('$out/ab_async_$1${mode}.json').read().strip().splitlines()[-1])
print('$1', '${mode:-sync}', b['value'], b['ms_per_step'], b['phases_ms'])" >> $out/ab_async.txt
  done
done
