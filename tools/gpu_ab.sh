O=gpurun_out/r02r
mkdir -p $O
for v in u2 u3; do
  timeout 900 python tools/ab_libs.py C4amg 2664 ab_libs/libvqpc_u4.so ab_libs/libvqpc_$v.so 1 > $O/ab_amg_$v.log 2>&1
  tail -n 2 $O/ab_amg_$v.log | head -1; tail -n 1 $O/ab_amg_$v.log
done
