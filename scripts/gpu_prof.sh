set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-analysis > gpurun_out/b_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_decode -s 3 -c 1 -o gpurun_out/kdec python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-analysis > gpurun_out/kdec.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stages -s 3 -c 1 -o gpurun_out/kst python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-analysis > gpurun_out/kst.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_an.csv python scripts/prof_analysis.py > gpurun_out/an_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_link_window|k_savings|k_als|k_dsd_demand" -c 8 -o gpurun_out/an python scripts/prof_analysis.py > gpurun_out/an_full.log 2>&1
ls -la gpurun_out
