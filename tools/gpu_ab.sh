O=gpurun_out/r02q
mkdir -p $O
for v in c1 c2; do
  timeout 900 python tools/ab_libs.py C4chol 2368 ab_libs/libvqpc_c0.so ab_libs/libvqpc_$v.so 1 > $O/ab_chol_$v.log 2>&1
  tail -n 2 $O/ab_chol_$v.log | head -1; tail -n 1 $O/ab_chol_$v.log
done
