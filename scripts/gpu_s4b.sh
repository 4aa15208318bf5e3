mkdir -p gpurun_out
timeout 600 python scripts/k1_harvest_probe.py "ES_K1_STAGE=full" "" "ES_K1_LPS=8" "ES_K1_LPS=32" > gpurun_out/s4b_probe.txt 2>&1
ES_K1_LPS=8 NSCEN=128 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_score -s 3 -c 1 \
  -o gpurun_out/s4b_k1h python scripts/k1_harvest_probe.py "" > /dev/null 2>&1
cat gpurun_out/s4b_probe.txt
