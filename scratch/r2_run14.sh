timeout 900 python -m pytest tests/test_harness.py -q -x 2>&1 | tail -15 > gpurun_out/r2_harness.log
timeout 600 python bench.py --config cadence --steps 300 --warmup 3 > gpurun_out/r2_bench_cadence.log 2>&1
timeout 600 python bench.py --config cadence --impl reference --steps 5 --warmup 1 > gpurun_out/r2_bench_cadence_ref.log 2>&1
