# One GPU session's measurements (run under gpurun from the repo root):
#   the GPU test suite, smoke, the microbenchmarked latencies, the bench line for
#   configs 4 / 5 / 7 and the reference arm, the ncu launch list of the bench step, and
#   --set full captures of the dominant kernel (k_decode, config 4) and of the config-5
#   prologue kernels (k_dsd_family, k_stages, the fill and clone passes, k_finalize),
#   k_relax alone on config 4's chain 33 (scripts/relax_solo.py --quiet), and the k_relax A/B.
# Other GPU scripts: gpu_ab.sh (same-box A/B of build/ab variants), gpu_sanitize.sh
# (compute-sanitizer over every entry point).
# Everything lands in gpurun_out/ with the prefix $TAG (e.g. r02c).
set -x
TAG=${TAG:-run}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest_gpu.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat scripts/ubench/lat.cu && /tmp/lat > gpurun_out/${TAG}_lat.txt 2>&1
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python bench.py --config 5 --steps 5 > gpurun_out/${TAG}_bench_cfg5.json 2> gpurun_out/${TAG}_bench_cfg5.err
python bench.py --config 7 --steps 10 > gpurun_out/${TAG}_bench_cfg7.json 2> gpurun_out/${TAG}_bench_cfg7.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-analysis > gpurun_out/${TAG}_b_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_decode -s 3 -c 1 -f -o gpurun_out/${TAG}_kdec python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-analysis > gpurun_out/${TAG}_kdec.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_dsd_family|k_stages|k_stage_clone|k_finalize" -s 5 -c 5 -f -o gpurun_out/${TAG}_cfg5pro python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-analysis > gpurun_out/${TAG}_cfg5pro.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_relax$" --launch-skip 1 -c 1 -f -o gpurun_out/${TAG}_krelax python scripts/relax_solo.py 0.73,0.74 --quiet > gpurun_out/${TAG}_krelax.log 2>&1
for c in 4 3 7; do timeout 400 python scripts/relax_ab.py $c 3; done > gpurun_out/${TAG}_relax_ab.txt 2>&1
ls -la gpurun_out
