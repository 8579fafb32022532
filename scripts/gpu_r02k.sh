# r02k: deferred DSD demand (k_stages beside k_dsd_family), family grid = one wave
set -x
TAG=${TAG:-r02k}
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "families or config2 or config5 or stage_groups or schedule or config4_reduced or random or edge or caps" > gpurun_out/${TAG}_tests.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_tests.log
timeout 600 python scripts/sched_times.py 5 > gpurun_out/${TAG}_cfg5_times.txt 2>&1
timeout 300 python scripts/sched_times.py 4 > gpurun_out/${TAG}_cfg4_times.txt 2>&1
