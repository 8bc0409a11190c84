# which earlier test file makes test_config4_shape_reduced_n flaky?
for combo in "tests/test_gpu_concurrency.py tests/test_gpu_dropin.py tests/test_gpu_fp32.py" "tests/test_gpu_kernels.py tests/test_gpu_ozaki.py tests/test_gpu_ozaki_syrk.py"; do
  for i in 1 2 3; do
    timeout 600 python -m pytest $combo tests/test_gpu_parity.py -q -p no:cacheprovider -k "not full_size" > gpurun_out/fc.log 2>&1
    echo "$combo rep $i: $(grep -E 'passed|failed' gpurun_out/fc.log | tail -1) $(grep -E '^E  .*assert' gpurun_out/fc.log | head -1)"
  done
done
