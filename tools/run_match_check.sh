mkdir -p gpurun_out
if [ "$1" != "quick" ]; then
timeout 900 python -m pytest tests/test_gpu_colcand.py tests/test_gpu_match_batch.py tests/test_gpu_parity.py tests/test_gpu_c4.py tests/test_gpu_pairs.py tests/test_gpu_ratio.py -m gpu -q > gpurun_out/g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g_tests.log
fi
timeout 300 python tools/tc_dense.py > gpurun_out/g_dense.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g_dense_launches.csv python tools/tc_dense.py > gpurun_out/g_ncu.log 2>&1
tail -3 gpurun_out/g_tests.log; tail -1 gpurun_out/g_dense.log; grep nn_topk_tc gpurun_out/g_dense_launches.csv | tail -2 | cut -c1-60,200-
