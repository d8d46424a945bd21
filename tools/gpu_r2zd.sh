S=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $S --tool racecheck --racecheck-report hazard --print-limit 8 python tools/run_once.py '{"kind":"conv2d","I":[2,64,14,18],"K":[64,64,3,3],"S":1}' tc_tf32 2>&1 | grep -v "^=========     #\|^========= *$" | head -60
