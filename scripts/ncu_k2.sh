# one ncu --set full capture of K2 per LPS setting (short bench run, 1 GPU)
for L in ${LPS_LIST:-16 32}; do
  ES_LPS=$L timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_replay -s 1 -c 1 \
    -o gpurun_out/prof_k2_lps$L python bench.py --steps 1 --warmup 1 --ncu > gpurun_out/ncu_lps$L.log 2>&1
  tail -2 gpurun_out/ncu_lps$L.log
done
