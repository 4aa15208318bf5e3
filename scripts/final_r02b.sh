# round-2 refresh after the K3 rework: smoke, GPU suite, bench line, launch list, ncu of K3 and the level pass
mkdir -p gpurun_out
R=${R:-r02k}
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$R.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -5 > gpurun_out/tests_$R.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
  python bench.py --steps 2 --warmup 1 --ncu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:k3_stats|k_group_level' -s 1 -c 2 \
  -o gpurun_out/prof_k3_$R python scripts/k3_time.py cfg3 > /dev/null 2>&1
tail -2 gpurun_out/smoke_$R.log; cat gpurun_out/tests_$R.log; tail -3 gpurun_out/bench_$R.err
