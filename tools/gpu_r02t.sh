# DRAM bytes per PCG launch (the roofline lines' `traffic`), final round-2 build
set -x
O=gpurun_out/r02t
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 900 $NCU --metrics $M --clock-control none -k regex:pcg2d -c 1 --csv --log-file $O/dram_c4.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > $O/ncu_dram_c4.log 2>&1
timeout 900 $NCU --metrics $M --clock-control none -k regex:pcgamg2d -c 1 --csv --log-file $O/dram_c4amg.csv \
  python bench.py --config C4amg --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > $O/ncu_dram_c4amg.log 2>&1
timeout 900 $NCU --metrics $M --clock-control none -k regex:pcgchol2d -c 1 --csv --log-file $O/dram_c4chol.csv \
  python bench.py --config C4chol --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > $O/ncu_dram_c4chol.log 2>&1
tail -n 4 $O/dram_*.csv
