# the failing condition of tools/gpu_flake3.sh with the DMMA mirrored SYRK's staged epilogue switched off
# (PSD_STAGED_EPI=0: direct mirrored stores from the accumulators)
O=gpurun_out/flake4; mkdir -p $O
for i in 1 2 3 4 5 6 7 8 9 10 11 12; do
  PSD_STAGED_EPI=0 PSD_CHOL_PIVOT=f timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "not full_size_fp64" -rf > $O/run_$i.log 2>&1; echo "rc=$?" >> $O/run_$i.log
  tail -2 $O/run_$i.log | head -1
done
grep -h "config4 shape\|FAILED" $O/*.log | head -20
