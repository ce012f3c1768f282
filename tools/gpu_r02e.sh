set -x
O=gpurun_out/r02e
mkdir -p $O
timeout 900 python -m pytest tests/test_amg.py tests/test_gpu_klbasis.py -q -s > $O/tests.log 2>&1
for S in 1 2 4; do VQPC_AMG_S=$S timeout 600 python tools/c4_modes.py C4amg 1024 > $O/amg_S$S.log 2>&1; done
bash tools/checks_build.sh > $O/checks.log 2>&1
tail -n 3 $O/*.log
