set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat scripts/ubench/lat.cu && /tmp/lat > gpurun_out/r02d_lat.txt 2>&1
/tmp/lat >> gpurun_out/r02d_lat_repeat.txt 2>&1
timeout 600 python scripts/chain_times.py 5 --no-walk > gpurun_out/r02d_cfg5_chain_times.txt 2>&1
