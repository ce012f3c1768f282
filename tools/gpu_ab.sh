O=gpurun_out/r02t
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "2d or ic0 or c4 or other_mesh" > $O/tests_2d.log 2>&1
tail -n 2 $O/tests_2d.log
timeout 900 python tools/ab_libs.py C4 2048 ab_libs/libvqpc_base.so paper_2403_07824_b200/libvqpc.so 1 > $O/ab_gmap.log 2>&1
tail -n 3 $O/ab_gmap.log
