#!/bin/bash
# window conv vs im2col TMA conv (both with the warp-collective MMA issue), CUDA events
run() { echo "$1 :: $(env $1 timeout 120 python scripts/conv_bench.py $2 20 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("%.1f us %.0f TF/s" % (d["ms"]*1e3, d["tflops"]))')"; }
for c in "256 56 56 64 64 3 3 1 1 fwd" "256 56 56 64 64 3 3 1 1 dgrad" "256 28 28 128 128 3 3 1 1 fwd" "256 28 28 128 128 3 3 1 1 dgrad" "256 14 14 256 256 3 3 1 1 fwd" "256 14 14 256 256 3 3 1 1 dgrad" "256 7 7 512 512 3 3 1 1 fwd"; do
  echo "== $c"
  run "TCB_WIN=0" "$c"
  run "TCB_WIN=1" "$c"
  run "TCB_WIN_CTA2=0" "$c"
done
