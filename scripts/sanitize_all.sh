# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over scripts/sanitize_cases.py
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool" >> gpurun_out/san_${R:-r02}.txt
  timeout 1200 compute-sanitizer --tool $tool --show-backtrace no --print-limit 10 python scripts/sanitize_cases.py \
    2>&1 | grep -v "Host Frame" | tail -16 >> gpurun_out/san_${R:-r02}.txt
done
cat gpurun_out/san_${R:-r02}.txt
