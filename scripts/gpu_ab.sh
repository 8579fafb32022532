# Same-box A/B of build/ab/<variant>.so kernels: parity first (every request of the
# GPU parity suite), then per-chain decode times for config 4 and config 5's slowest
# chains.  usage (under gpurun): TAG=... bash scripts/gpu_ab.sh base v1 v2 ...
TAG=${TAG:-ab}
for n in "$@"; do
  if [ "$n" != base ]; then
    GL_LIB_PATH=build/ab/$n.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${TAG}_${n}_parity.log 2>&1
    echo "$n parity exit $?" >> gpurun_out/${TAG}_summary.txt
  fi
done
for rep in 1 2; do
  for n in "$@"; do
    echo "== $n (rep $rep)" >> gpurun_out/${TAG}_times.txt
    GL_LIB_PATH=build/ab/$n.so CHAINS=${CHAINS:-33,51,46,36} python scripts/quick_times.py ${CHAINS:-33,51,46,36} 4 >> gpurun_out/${TAG}_times.txt 2>&1
    GL_LIB_PATH=build/ab/$n.so python scripts/quick_times.py ${CHAINS5:-34,33,319} 5 >> gpurun_out/${TAG}_times.txt 2>&1
  done
done
