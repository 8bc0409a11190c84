# hunt for the intermittent C4-shape failure: the GPU suite without the two full-size C3 cases,
# alternating the env that was set when it last failed; full failure output kept
O=gpurun_out/flake2; mkdir -p $O
for i in 1 2 3 4 5; do for V in f d; do
  PSD_CHOL_PIVOT=$V timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "not full_size_fp64" -rf > $O/run_${V}_$i.log 2>&1; echo "rc=$?" >> $O/run_${V}_$i.log
  tail -2 $O/run_${V}_$i.log | head -1
done; done
grep -h "config4 shape\|FAILED" $O/*.log | head -20
