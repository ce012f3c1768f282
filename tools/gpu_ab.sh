O=gpurun_out/r02o
mkdir -p $O
VQPC_LIB=ab_libs/libvqpc_base.so timeout 900 python bench.py --config C4amg --steps 2 --warmup 2 --no-cpu --e2e-steps 1 > $O/bench_c4amg_baselib.json 2> $O/bench_c4amg_baselib.err
tail -c 300 $O/bench_c4amg_baselib.json
timeout 900 python bench.py --config C4amg --steps 2 --warmup 2 --no-cpu --e2e-steps 1 > $O/bench_c4amg_newlib.json 2> $O/bench_c4amg_newlib.err
