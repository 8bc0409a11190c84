# round 2: full GPU suite (incl. full-size C3 parity) + short bench
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > gpurun_out/pytest_r2b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2b.log
tail -30 gpurun_out/pytest_r2b.log
