O=gpurun_out/r02u
mkdir -p $O
timeout 1500 python -m pytest tests/test_amg.py tests/test_ideal_sweep.py tests/test_integration.py tests/test_gpu_edges.py -q -m gpu > $O/amg_tests_s2.log 2>&1
tail -n 2 $O/amg_tests_s2.log
timeout 1200 python bench.py --config C4amg --steps 3 --warmup 3 > $O/bench_c4amg_s2.json 2> $O/bench_c4amg_s2.err
tail -c 100 $O/bench_c4amg_s2.json
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_s2.log 2>&1
tail -n 2 $O/smoke_s2.log
