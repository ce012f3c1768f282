set -x
mkdir -p gpurun_out/r02b
timeout 900 python -m pytest tests/test_amg.py tests/test_integration.py -q -s > gpurun_out/r02b/amg_tests.log 2>&1
timeout 600 python tools/c4_modes.py C4amg 1024 > gpurun_out/r02b/c4amg_modes.log 2>&1
timeout 900 python bench.py --config C4amg --steps 2 --warmup 1 --no-cpu > gpurun_out/r02b/bench_c4amg.json 2> gpurun_out/r02b/bench_c4amg.err
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -s > gpurun_out/r02b/fullsize.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --ignore tests/test_gpu_fullsize.py --ignore tests/test_amg.py --ignore tests/test_integration.py > gpurun_out/r02b/gputests.log 2>&1
tail -3 gpurun_out/r02b/*.log
