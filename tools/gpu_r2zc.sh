mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2zc_pytest_gpu.log 2>&1; tail -3 gpurun_out/r2zc_pytest_gpu.log
S=/usr/local/cuda/bin/compute-sanitizer
for op in '{"kind":"conv2d","I":[2,64,14,18],"K":[64,64,3,3],"S":1}' '{"kind":"conv2d","I":[3,32,8,12],"K":[64,32,3,3],"S":1}'; do
  timeout 600 $S --tool memcheck python tools/run_once.py "$op" tc_tf32 2>&1 | grep -E "ERROR SUMMARY|cta_pair" | sed 's/.*"cta_pair": \([a-z]*\).*/cta_pair=\1/'
  timeout 900 $S --tool racecheck --racecheck-report hazard python tools/run_once.py "$op" tc_tf32 2>&1 | grep -E "RACECHECK SUMMARY"
  timeout 900 $S --tool synccheck python tools/run_once.py "$op" tc_tf32 2>&1 | grep -E "ERROR SUMMARY"
done
