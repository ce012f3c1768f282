O=gpurun_out/r02w
mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -k "not 2d and not ic0 and not c4 and not other_mesh" > $O/tests_1d.log 2>&1
tail -n 2 $O/tests_1d.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -n 3 $O/smoke.log
timeout 600 python bench.py --config C1 --steps 3000 --warmup 20 > $O/bench_c1.json 2> $O/bench_c1.err
