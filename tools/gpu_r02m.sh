# ncu source-level capture of the SA-AMG PCG kernel (C4amg, 444 samples = 3 CTAs per SM once)
set -x
O=gpurun_out/r02m
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 600 python bench.py --config C4amg --n 444 --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > $O/plain.log 2>&1 || exit 1
timeout 1500 $NCU --section SourceCounters --section WarpStateStats --section SchedulerStats --section MemoryWorkloadAnalysis --section SpeedOfLight --section Occupancy --section LaunchStats --clock-control none --import-source on -k regex:pcgamg2d -c 1 -f -o $O/pcgamg2d_444 \
  python bench.py --config C4amg --n 444 --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > $O/ncu.log 2>&1
tail -3 $O/ncu.log
