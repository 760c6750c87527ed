TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
out=gpurun_out; mkdir -p $out
for v in a b; do
timeout 600 $TR --nproc-per-node 4 --master-port 2961$((RANDOM%9)) bench.py --gpus 4 --no-cpu-baseline --no-e2e > $out/r01v_g4_overlap_$v.json 2> $out/r01v_g4_overlap_$v.err
timeout 600 $TR --nproc-per-node 4 --master-port 2962$((RANDOM%9)) bench.py --gpus 4 --no-cpu-baseline --no-e2e --no-overlap > $out/r01v_g4_nooverlap_$v.json 2> $out/r01v_g4_nooverlap_$v.err
done
timeout 600 $TR --nproc-per-node 2 --master-port 29631 bench.py --gpus 2 --no-cpu-baseline > $out/r01v_g2.json 2> $out/r01v_g2.err
