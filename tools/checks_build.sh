# The check build: libvqpc_checks.so with device-side bounds/invariant checks
# (VQPC_DCHECK, common.cuh), then the GPU parity tests against it. Usage on a GPU box:
#   bash tools/checks_build.sh [pytest -k expression]
set -e
VQPC_LIB=$PWD/paper_2403_07824_b200/libvqpc_checks.so VQPC_NVCC_FLAGS="-DVQPC_CHECKS" \
  python -c "from paper_2403_07824_b200 import build; build.build(force=True)"
VQPC_LIB=$PWD/paper_2403_07824_b200/libvqpc_checks.so python -m pytest tests -m gpu -q -x \
  --ignore tests/test_gpu_fullsize.py ${1:+-k "$1"}
