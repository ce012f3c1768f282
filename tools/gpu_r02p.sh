# the check build (VQPC_DCHECK device assertions) against the GPU suite, final round-2 code
set -x
O=gpurun_out/r02p
mkdir -p $O
timeout 3000 bash tools/checks_build.sh > $O/checks.log 2>&1
tail -n 4 $O/checks.log
VQPC_LIB=$PWD/paper_2403_07824_b200/libvqpc_checks.so timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -k "paper_size or c4_full_size_exact" >> $O/checks.log 2>&1
tail -n 2 $O/checks.log
