# last lease of the round: three more full GPU suites (flake hunt), the headline bench line on the
# final bench.py (pipelined + unpipelined values) and the ncu capture of the symmetric α-estimate kernel
O=gpurun_out/fin; mkdir -p $O
for i in 1 2 3; do
  timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/suite$i.log 2>&1; echo "rc=$?" >> $O/suite$i.log
done
timeout 900 python bench.py --steps 16 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:symv_tiles -s 2 -c 1 -o $O/full_symv_tiles python bench.py --steps 1 --warmup 1 --pool 1 --no-peaks --no-e2e --no-cpu-baseline --no-c4 --no-fp32 > $O/ncu_full_symv.log 2>&1
tail -n 2 $O/suite*.log; cut -c1-300 $O/bench_c3.json
