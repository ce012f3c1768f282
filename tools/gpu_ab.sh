O=gpurun_out/r02q
mkdir -p $O
for v in pf1 pf2 pf3 pf2l1; do
  timeout 900 python tools/ab_libs.py C4amg 2664 ab_libs/libvqpc_pf0.so ab_libs/libvqpc_$v.so 1 > $O/ab_amg2_$v.log 2>&1
  tail -n 2 $O/ab_amg2_$v.log | head -1; tail -n 1 $O/ab_amg2_$v.log
done
