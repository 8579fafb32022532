# r02h: two-phase launch order (gl_schedule): its GPU test first, the full GPU suite,
# schedule on/off device times for configs 4 / 5 / 3, bench configs 4 / 5
set -x
TAG=${TAG:-r02h}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k schedule > gpurun_out/${TAG}_sched_test.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_sched_test.log
timeout 600 python scripts/sched_times.py 4 5 3 > gpurun_out/${TAG}_sched_times.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest_gpu.log
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python bench.py --config 5 --steps 5 > gpurun_out/${TAG}_bench_cfg5.json 2> gpurun_out/${TAG}_bench_cfg5.err
