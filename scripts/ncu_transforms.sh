#!/bin/bash
# ncu --set full of the Winograd / FFT transform kernels on AlexNet conv3 (bs256)
out=gpurun_out; tag=${1:-r02t}
for algo in fft winograd; do
  timeout 120 python scripts/conv_bench.py 256 13 13 256 384 3 3 1 1 fwd 3 $algo bf16 > $out/${tag}_${algo}_plain.log 2>&1 || { echo plain failed; exit 1; }
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fft_fwd_smem|fft_inv_smem|wino_input_smem|wino_output" -c 2 \
    -o /tmp/${tag}_${algo} -f python scripts/conv_bench.py 256 13 13 256 384 3 3 1 1 fwd 1 $algo bf16 > $out/${tag}_${algo}_ncu.log 2>&1
  ncu -i /tmp/${tag}_${algo}.ncu-rep --page details --csv > $out/${tag}_${algo}_details.csv 2>> $out/${tag}_${algo}_ncu.log
  ncu -i /tmp/${tag}_${algo}.ncu-rep --page raw --csv > $out/${tag}_${algo}_raw.csv 2>> $out/${tag}_${algo}_ncu.log
done
echo done
