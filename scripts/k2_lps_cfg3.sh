for L in 32 16 8; do
  ES_K2_MAP=seg ES_LPS=$L timeout 300 python bench.py --workload cfg3 --steps 2 --warmup 3 --no-k1 --no-e2e --no-cpu-baseline > gpurun_out/sw.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sw.json')); print('lps $L k2_ms', round(d['roofline']['k2_ms'],2), 'dec/s %.3e'%d['value'])"
done
