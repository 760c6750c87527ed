#!/bin/bash
# Round-2 multi-GPU evidence on one 4-GPU box: PS tests, bench at 1 / 2 / 4 GPUs
# (NVLS PS step) and the NCCL PS step at 4 GPUs.
#   gpurun --gpus 4 --timeout 2400 -- bash scripts/r02_multi.sh
out=gpurun_out
timeout 900 python -m pytest tests/test_ps_multigpu.py -m gpu -q -p no:cacheprovider > $out/r02h_ps_multigpu_g4.log 2>&1
for g in 1 2 4; do
  if [ $g = 1 ]; then
    timeout 600 python bench.py > $out/r02h_scale_g$g.json 2> $out/r02h_scale_g$g.err
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 \
      --master-port 29611 bench.py --gpus $g > $out/r02h_scale_g$g.json 2> $out/r02h_scale_g$g.err
  fi
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29612 bench.py --gpus 4 --ps-transport nccl > $out/r02h_scale_g4_nccl.json 2> $out/r02h_scale_g4_nccl.err
tail -2 $out/r02h_ps_multigpu_g4.log
for f in $out/r02h_scale_g1.json $out/r02h_scale_g2.json $out/r02h_scale_g4.json $out/r02h_scale_g4_nccl.json; do
  python -c "import json,sys; b=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', b['value'], b['ms_per_step'], b['e2e']['value'], b.get('phases_ms'))"
done
