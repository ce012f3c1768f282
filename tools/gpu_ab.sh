O=gpurun_out/r02q
mkdir -p $O
timeout 1200 python -m pytest tests/test_amg.py tests/test_ideal_sweep.py tests/test_integration.py -q -m gpu > $O/amg_tests.log 2>&1
tail -n 2 $O/amg_tests.log
timeout 1200 python bench.py --config C4amg --steps 3 --warmup 3 > $O/bench_c4amg.json 2> $O/bench_c4amg.err
tail -c 200 $O/bench_c4amg.json
