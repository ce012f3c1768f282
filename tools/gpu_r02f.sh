# C4 (default) bench as the driver runs it, the reference arm, and the ncu evidence
set -x
O=gpurun_out/r02f
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
date +%s > $O/t0; timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench_c4.json 2> $O/bench_c4.err; date +%s > $O/t1
NCU=/usr/local/cuda/bin/ncu
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > $O/ncu_launch.log 2>&1
timeout 900 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:pcg2d -c 1 --csv --log-file $O/dram_c4.csv python bench.py --steps 1 --warmup 1 --no-cpu --e2e-steps 1 \
  > $O/ncu_dram.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:pcg2d -c 1 -o $O/pcg2d_c4_592 \
  python bench.py --n 592 --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > $O/ncu_full.log 2>&1
python tools/ab_libs.py C4amg 1024 paper_2403_07824_b200/libvqpc.so paper_2403_07824_b200/libvqpc_u2.so > $O/ab_amg_u2.log 2>&1
python tools/ab_libs.py C4amg 1024 paper_2403_07824_b200/libvqpc.so paper_2403_07824_b200/libvqpc_m3.so > $O/ab_amg_m3.log 2>&1
python tools/ab_libs.py C4amg 1024 paper_2403_07824_b200/libvqpc.so paper_2403_07824_b200/libvqpc_u2m3.so > $O/ab_amg_u2m3.log 2>&1
tail -n 3 $O/*.log $O/*.err
