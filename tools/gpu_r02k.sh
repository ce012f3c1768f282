# round-2 (third session): full GPU suite on the committed build, then every config's bench line
set -x
O=gpurun_out/r02k
mkdir -p $O
timeout 3000 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1
tail -n 5 $O/gpu_tests.log
for c in C1 C2 C3 C5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
  tail -c 600 $O/bench_$c.json
done
