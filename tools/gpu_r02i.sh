set -x
O=gpurun_out/r02i
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:pcgamg2d -c 1 -o $O/pcgamg2d_444 \
  python bench.py --config C4amg --n 444 --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > $O/ncu_full.log 2>&1
tail -n 4 $O/*.log
timeout 900 python tools/ab_env.py C4 8192 VQPC_P2_PAIR=0 VQPC_P2_PAIR=1 1 > $O/ab_pair_c4_8192.log 2>&1
timeout 900 python -m pytest tests/test_amg.py -q -x > $O/amg_tests.log 2>&1
timeout 600 python tools/c4_modes.py C4amg 1024 > $O/amg_structured.log 2>&1
tail -n 4 $O/*.log
