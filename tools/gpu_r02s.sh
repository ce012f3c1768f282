# round-2 final evidence on the committed build: full GPU suite, smoke, the default bench as the
# driver runs it, the reference arm, C4amg / C4chol / C2 lines, and the ncu launch list
set -x
O=gpurun_out/r02s
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1
tail -n 3 $O/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
tail -n 3 $O/smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench_c4.json 2> $O/bench_c4.err
tail -c 400 $O/bench_c4.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_c4_reference.json 2> $O/bench_c4_reference.err
timeout 1200 python bench.py --config C4amg --steps 3 --warmup 3 > $O/bench_c4amg.json 2> $O/bench_c4amg.err
timeout 1200 python bench.py --config C4chol --steps 3 --warmup 3 --no-cpu > $O/bench_c4chol.json 2> $O/bench_c4chol.err
timeout 900 python bench.py --config C2 --steps 10 --warmup 3 > $O/bench_c2.json 2> $O/bench_c2.err

NCU=/usr/local/cuda/bin/ncu
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > $O/ncu_launch.log 2>&1
tail -n 2 $O/*.err
