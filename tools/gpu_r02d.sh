set -x
O=gpurun_out/r02d
mkdir -p $O
timeout 900 python tools/make_artifacts.py C5 C4 > $O/arts.log 2>&1
timeout 1500 python -m pytest tests/test_amg.py tests/test_ideal_sweep.py tests/test_gpu_klbasis.py -q -s > $O/tests.log 2>&1
for S in 1 2 4 8; do VQPC_AMG_S=$S timeout 600 python tools/c4_modes.py C4amg 1024 > $O/amg_S$S.log 2>&1; done
tail -n 3 $O/*.log
