# Round artefacts: GPU tests, full bench line, ncu launch list, one ncu --set full
# capture each of K2, K3 and the K1 call (bench-size batch), the reference arm
R=${R:-r01}
timeout 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -3 > gpurun_out/tests_$R.log
timeout 400 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
tail -2 gpurun_out/bench_$R.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
  python bench.py --steps 2 --warmup 1 --ncu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_replay -s 1 -c 1 \
  -o gpurun_out/prof_k2_$R python bench.py --steps 1 --warmup 1 --ncu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k3_stats -s 1 -c 1 \
  -o gpurun_out/prof_k3_$R python bench.py --steps 1 --warmup 1 --ncu > /dev/null 2>&1
K1_BIG=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1s_ -s 4 -c 4 \
  -o gpurun_out/prof_k1_$R python scripts/k1_probe.py stream > /dev/null 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$R.json 2>&1
cat gpurun_out/tests_$R.log
ls gpurun_out
