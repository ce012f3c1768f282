set -x
O=gpurun_out/r02c
mkdir -p $O
timeout 600 python tools/make_artifacts.py C5 C4 > $O/arts.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_chol2d.py tests/test_ideal_sweep.py tests/test_gpu_klbasis.py tests/test_amg.py -q -s > $O/new_tests.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -s -k "C5 or c4_full_size_256" > $O/fullsize.log 2>&1
bash tools/sanitize_all.sh $O/sanitize > $O/sanitize_run.log 2>&1
tail -3 $O/*.log; cat $O/sanitize/summary.txt
