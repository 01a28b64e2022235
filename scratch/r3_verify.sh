mkdir -p gpurun_out/v
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/v/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/v/bench_c3.log 2>&1
timeout 900 python bench.py --config cadence --steps 300 --warmup 3 > gpurun_out/v/bench_cad.log 2>&1
