# r02g: GPU tests (k_stage_clone 4-wide, k_finalize unrolled), bench configs 4 / 5 / 7, launch list
set -x
TAG=${TAG:-r02g}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest_gpu.log
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python bench.py --config 5 --steps 5 > gpurun_out/${TAG}_bench_cfg5.json 2> gpurun_out/${TAG}_bench_cfg5.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_stage_clone|k_finalize|k_stages|k_dsd" -c 12 --csv --log-file gpurun_out/${TAG}_cfg5_prologue.csv python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-analysis > gpurun_out/${TAG}_cfg5_ncu.log 2>&1
