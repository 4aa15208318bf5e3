# round 2 (d): GPU tests, bench with the K1 clip/harvested lines, policy table
# from the group counters, compute-sanitizer over every kernel family
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02d_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -25 > gpurun_out/r02d_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err
timeout 600 python scripts/policy_table.py > gpurun_out/r02d_policies.txt 2> gpurun_out/r02d_policies.err
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/r02d_san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r02d_san_rc.txt
done
tail -3 gpurun_out/r02d_smoke.log; tail -5 gpurun_out/r02d_tests.log; cat gpurun_out/r02d_san_rc.txt; tail -c 1500 gpurun_out/r02d_bench.json
