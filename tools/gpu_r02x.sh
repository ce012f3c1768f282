# ncu --set full of the final pcg2d (IC(0)) kernel: one wave of 592 samples (two CTAs per SM)
set -x
O=gpurun_out/r02x
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 600 python bench.py --n 592 --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > $O/plain.log 2>&1 || exit 1
timeout 1500 $NCU --set full --clock-control none --import-source on -k regex:pcg2d -c 1 -f -o $O/pcg2d_c4_592 \
  python bench.py --n 592 --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > $O/ncu_full.log 2>&1
tail -2 $O/ncu_full.log
