#!/bin/bash
# A/B of the window conv's knobs on the ResNet-50 3x3 layers (bs256), CUDA events.
run() { echo "$1 :: $(env $1 timeout 120 python scripts/conv_bench.py $2 20 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("%.1f us %.0f TF/s" % (d["ms"]*1e3, d["tflops"]))')"; }
for c in "256 56 56 64 64 3 3 1 1 fwd" "256 28 28 128 128 3 3 1 1 fwd" "256 28 28 128 128 3 3 1 1 dgrad"; do
  echo "== $c"
  run "TCB_WIN=0" "$c"
  run "TCB_WIN=1" "$c"
  run "TCB_WIN_CTA2=0" "$c"
  run "TCB_WIN_BRES=0" "$c"
  run "TCB_WIN_WSTAGES=2" "$c"
  run "TCB_WIN_WSTAGES=2 TCB_WIN_BSTAGES=8" "$c"
  run "TCB_WIN_BSTAGES=4" "$c"
done
