O=gpurun_out/r02m
mkdir -p $O
for c in "C5 16384" "C2 32768" "C4 1024"; do
  timeout 600 python tools/realise_ab.py $c ab_libs/libvqpc_base.so paper_2403_07824_b200/libvqpc.so >> $O/ab_realise.log 2>&1
done
cat $O/ab_realise.log | grep -v "^$" | tail -9
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "realise or exact_mode_campaign" > $O/realise_tests.log 2>&1
tail -n 2 $O/realise_tests.log
