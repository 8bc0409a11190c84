# after the fence fix: the condition that failed 2 of 6 times (suite without the full-size cases, PSD_CHOL_PIVOT=f)
O=gpurun_out/flake3; mkdir -p $O
for i in 1 2 3 4 5 6 7 8; do
  PSD_CHOL_PIVOT=f timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "not full_size_fp64" -rf > $O/run_$i.log 2>&1; echo "rc=$?" >> $O/run_$i.log
  tail -2 $O/run_$i.log | head -1
done
grep -h "config4 shape\|FAILED" $O/*.log | head -20
