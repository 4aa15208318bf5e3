timeout 1500 python scripts/k2_width_sweep.py ${ARGS:-cfg2:8,16 cfg3:16,32 cfg5a:16,32 cfg5b:16,32 cfg4:8,16} 2>&1 | grep -v Warning
