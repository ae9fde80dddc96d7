mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/f_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/f_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/f_bench.log 2> gpurun_out/f_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/f_launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-match --no-stitch --no-pairs --no-composite > gpurun_out/f_ncu1.log 2>&1
timeout 900 ncu -k regex:describe_f32_tile_kernel --launch-skip 1 --launch-count 1 --set full --import-source on --clock-control none -o gpurun_out/f_describe -f python bench.py --profile-steps 2 --no-cpu --no-e2e --no-match --no-stitch --no-pairs --no-composite > gpurun_out/f_ncu2.log 2>&1
ncu -i gpurun_out/f_describe.ncu-rep --page raw --csv > gpurun_out/f_describe_raw.csv 2>/dev/null
ncu -i gpurun_out/f_describe.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/f_describe_src.csv 2>/dev/null
tail -2 gpurun_out/f_tests.log; tail -1 gpurun_out/f_smoke.log; ls -la gpurun_out/f_*
# the dense tensor-core match: launch list and one full capture of the top-k pass
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches_dense.csv python tools/tc_dense.py > gpurun_out/f_ncu3.log 2>&1
timeout 600 ncu -k regex:nn_topk_tc --launch-skip 2 --launch-count 1 --set full --import-source on --clock-control none -o gpurun_out/f_topk -f python tools/tc_dense.py > gpurun_out/f_ncu4.log 2>&1
ncu -i gpurun_out/f_topk.ncu-rep --page raw --csv > gpurun_out/f_topk_raw.csv 2>/dev/null
# the strip detectors (C4 L = 36, C5 RGB)
timeout 600 ncu -k regex:detect_strip --set full --import-source on --clock-control none -o gpurun_out/f_detect -f python tools/det_one.py > gpurun_out/f_ncu5.log 2>&1
ncu -i gpurun_out/f_detect.ncu-rep --page raw --csv > gpurun_out/f_detect_raw.csv 2>/dev/null
