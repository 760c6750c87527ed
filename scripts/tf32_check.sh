mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_trainer_gpu.py -m gpu -q -p no:cacheprovider -k "tf32" > gpurun_out/tf32_pytest.log 2>&1; echo rc=$? >> gpurun_out/tf32_pytest.log
timeout 400 python bench.py --precision tf32 --steps 5 --warmup 3 > gpurun_out/tf32_bench.json 2> gpurun_out/tf32_bench.err; echo rc=$? >> gpurun_out/tf32_bench.err
