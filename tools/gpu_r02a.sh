set -x
mkdir -p gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a/smi.txt
timeout 600 python tools/make_artifacts.py C5 > gpurun_out/r02a/arts.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r02a/bench_c4.json 2> gpurun_out/r02a/bench_c4.err
timeout 600 python tools/c4_modes.py C4 1024 > gpurun_out/r02a/c4_modes.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -x -q -s > gpurun_out/r02a/fullsize.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --deselect "tests/test_integration.py::test_adapter_report_equals_ctypes_run[C4s-48-amg-None]" --ignore tests/test_gpu_fullsize.py > gpurun_out/r02a/gputests.log 2>&1
tail -3 gpurun_out/r02a/*.log
