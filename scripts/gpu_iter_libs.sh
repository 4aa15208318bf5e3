# time the cfg3 K2 batch with several library builds (LIBS) and variants (VARIANTS)
mkdir -p gpurun_out; : > gpurun_out/iter_libs.txt
for lib in ${LIBS:-libedgeserve}; do
  echo "== $lib" >> gpurun_out/iter_libs.txt
  ES_LIB=$PWD/paper_2605_05527_b200/$lib.so timeout 600 python scripts/k2_mapping.py ${W:-cfg3} ${S:-65536} "${VARIANTS:--}" 2>&1 | grep K2 >> gpurun_out/iter_libs.txt
done
cat gpurun_out/iter_libs.txt
