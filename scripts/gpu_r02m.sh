# r02m: the round's measurement session after the prologue work (tests, smoke,
# bench configs 4 / 5 / 7, launch list, k_decode and config-5 prologue captures)
set -x
TAG=${TAG:-r02s}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest_gpu.log
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python bench.py --config 5 --steps 5 > gpurun_out/${TAG}_bench_cfg5.json 2> gpurun_out/${TAG}_bench_cfg5.err
python bench.py --config 7 --steps 10 > gpurun_out/${TAG}_bench_cfg7.json 2> gpurun_out/${TAG}_bench_cfg7.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-analysis > gpurun_out/${TAG}_b_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_decode -s 3 -c 1 -f -o gpurun_out/${TAG}_kdec python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-analysis > gpurun_out/${TAG}_kdec.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_dsd_family|k_stages|k_stage_clone|k_stage_fill|k_finalize" -s 5 -c 5 -f -o gpurun_out/${TAG}_cfg5pro python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-analysis > gpurun_out/${TAG}_cfg5pro.log 2>&1
ls -la gpurun_out
