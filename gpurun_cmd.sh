python -m pytest tests/test_kernels_gpu.py -x -q -k "fc_forward_split or vgg_fc or plain_1x1 or wgrad_many" 2>&1 | tail -15
python -m pytest tests/test_trainer_gpu.py tests/test_bench_configs_gpu.py -x -q 2>&1 | tail -15
python -m pytest tests/test_canaries_gpu.py tests/test_stem_gpu.py -x -q 2>&1 | tail -5
