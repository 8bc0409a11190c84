# repeated full GPU suites to catch the intermittent C4-shape parity failure
O=gpurun_out/flake; mkdir -p $O
for i in 1 2 3 4 5; do
  timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/run$i.log 2>&1; echo "rc=$?" >> $O/run$i.log
  tail -3 $O/run$i.log
done
grep -h "config4 shape\|FAILED\|rel err" $O/run*.log | head -40
