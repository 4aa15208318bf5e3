for v in ${VARIANTS:-v0 v1 v3}; do
  for r in 1 3; do echo -n "$v reps $r: "; ES_LIB=$PWD/variants/$v.so ES_LPS=16 timeout 60 python scripts/debug_lps.py $r 2>&1 | grep -E "^reps|Error" | head -1 | cut -c1-150; done
done
