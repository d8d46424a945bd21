set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout 900 python bench.py --workload gpt2 --steps 5 --warmup 3 > gpurun_out/bench_gpt2.log 2>&1
timeout 900 python bench.py --workload resnet50 --steps 3 --warmup 3 > gpurun_out/bench_resnet50.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
