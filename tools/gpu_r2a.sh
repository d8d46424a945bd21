# round-2 check: full GPU suite + default bench + smoke
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2a_pytest_gpu.log 2>&1
tail -30 gpurun_out/r2a_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1
tail -3 gpurun_out/r2a_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.jsonl 2> gpurun_out/r2a_bench.err
tail -c 3000 gpurun_out/r2a_bench.jsonl
