set -x
O=gpurun_out/r02h
mkdir -p $O
timeout 1200 python bench.py --config C4amg --steps 3 --warmup 3 > $O/bench_c4amg.json 2> $O/bench_c4amg.err
timeout 1200 python bench.py --config C4chol --steps 3 --warmup 3 --no-cpu > $O/bench_c4chol.json 2> $O/bench_c4chol.err
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
sed -i 's/ -x / /' tools/checks_build.sh
timeout 2400 bash tools/checks_build.sh > $O/checks.log 2>&1
tail -n 4 $O/*.log
