free -g > gpurun_out/r2x_free.txt 2>&1; nproc >> gpurun_out/r2x_free.txt
timeout 900 python -m pytest tests/test_async_gpu.py tests/test_forward_gpu.py tests/test_kernels_gpu.py -m gpu -q -k "swap or submit or pipelined" > gpurun_out/r2x_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2x_tests.log
AG_BENCH_TRACE=1 timeout -s ABRT 900 python -X faulthandler bench.py --rate 4 --steps 30 --no-cpu-baseline > gpurun_out/r2x_bench.jsonl 2> gpurun_out/r2x_bench.err; echo rc=$? >> gpurun_out/r2x_bench.err
