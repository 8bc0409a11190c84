# compute-sanitizer over every kernel family (tools/sanitize_run.py), reduced n
export PSD_OZ_SYRK=1
S=/usr/local/cuda/bin/compute-sanitizer
timeout 300 python tools/sanitize_run.py 3072 > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/san_plain.log
for T in memcheck synccheck racecheck; do
  timeout 1500 $S --tool $T --print-limit 50 --error-exitcode 9 python tools/sanitize_run.py 3072 > gpurun_out/san_$T.log 2>&1
  echo "$T rc=$?" >> gpurun_out/san_$T.log
done
tail -n 4 gpurun_out/san_*.log
