# the 512-thread IC(0) kernels (257 < r <= 513) and the limits
set -x
O=gpurun_out/r02l
mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_fullsize.py -q -x -k "other_mesh_sizes or size_limits or paper_size or 2d or ic0" -s > $O/tests_big_mesh.log 2>&1
tail -n 8 $O/tests_big_mesh.log
