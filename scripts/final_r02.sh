# final round-2 check on the current build: smoke, GPU suite, bench line, reference arm, ncu of the K1 calls
mkdir -p gpurun_out
R=${R:-r02f}
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$R.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -5 > gpurun_out/tests_$R.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$R.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:k1_thread|k1_score' -s 2 -c 2 \
  -o gpurun_out/prof_k1h_$R python scripts/k1_harvest_probe.py "" > /dev/null 2>&1
tail -2 gpurun_out/smoke_$R.log; cat gpurun_out/tests_$R.log; tail -3 gpurun_out/bench_$R.err
