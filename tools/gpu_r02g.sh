set -x
O=gpurun_out/r02g
mkdir -p $O
timeout 900 python tools/ab_env.py C4 2048 VQPC_P2_PAIR=0 VQPC_P2_PAIR=1 1 > $O/ab_pair_c4.log 2>&1
timeout 900 python tools/ab_env.py C4s 512 VQPC_P2_PAIR=0 VQPC_P2_PAIR=1 1 exact > $O/ab_pair_c4s_exact.log 2>&1
timeout 900 python tools/ab_env.py C4s 512 VQPC_P2_PAIR=0 VQPC_P2_PAIR=1 1 > $O/ab_pair_c4s.log 2>&1
timeout 600 python tools/c4_modes.py C4amg 1024 > $O/amg_m3.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_amg.py -q -x > $O/tests.log 2>&1
tail -n 4 $O/*.log
