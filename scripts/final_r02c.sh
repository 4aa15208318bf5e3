# last round-2 check on HEAD: smoke, GPU suite, bench line
mkdir -p gpurun_out
R=${R:-r02z}
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$R.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -5 > gpurun_out/tests_$R.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
tail -2 gpurun_out/smoke_$R.log; cat gpurun_out/tests_$R.log; tail -3 gpurun_out/bench_$R.err
