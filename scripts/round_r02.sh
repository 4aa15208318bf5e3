# Round-2 artefacts: smoke, GPU suite, bench line, launch list, ncu --set full of K2 / K3 / the
# three K1 calls (5-C stream, harvested cfg3, clip path), the reference arm, f1 policy table, f3 sweeps
mkdir -p gpurun_out
R=${R:-r02}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$R.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -5 > gpurun_out/tests_$R.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
  python bench.py --steps 2 --warmup 1 --ncu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_replay -s 1 -c 1 \
  -o gpurun_out/prof_k2_$R python bench.py --steps 1 --warmup 1 --ncu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k3_stats -s 1 -c 1 \
  -o gpurun_out/prof_k3_$R python bench.py --steps 1 --warmup 1 --ncu > /dev/null 2>&1
K1_BIG=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1s_ -s 4 -c 4 \
  -o gpurun_out/prof_k1_$R python scripts/k1_probe.py stream > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k1_thread|k1_score' -s 2 -c 2 \
  -o gpurun_out/prof_k1h_$R python scripts/k1_harvest_probe.py "" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1s_ -s 4 -c 4 \
  -o gpurun_out/prof_k1clip_$R python scripts/k1_clip_once.py 1 > /dev/null 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$R.json 2>&1


tail -2 gpurun_out/smoke_$R.log; cat gpurun_out/tests_$R.log; tail -3 gpurun_out/bench_$R.err
ls gpurun_out
