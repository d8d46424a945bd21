# round-2 re-entry: full GPU suite, smoke, default bench, ncu launch list of the default bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2k_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2k_pytest_gpu.log 2>&1
tail -15 gpurun_out/r2k_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k_smoke.log 2>&1
tail -3 gpurun_out/r2k_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2k_bench.jsonl 2> gpurun_out/r2k_bench.err
tail -3 gpurun_out/r2k_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2k_ref.jsonl 2> gpurun_out/r2k_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2k_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2k_ncu_bench.log 2>&1
echo done
