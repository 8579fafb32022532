# compute-sanitizer over every C-ABI entry point (scripts/sanitize_run.py)
TAG=${TAG:-san}
for tool in memcheck synccheck initcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 400 python scripts/sanitize_run.py > gpurun_out/${TAG}_${tool}.log 2>&1
  echo "exit $?" >> gpurun_out/${TAG}_${tool}.log
done
