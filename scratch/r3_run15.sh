mkdir -p gpurun_out/q
timeout 900 python -m pytest tests/test_gpu_graphs.py tests/test_gpu_pipeline.py tests/test_gpu_gates.py -q -m gpu > gpurun_out/q/t.log 2>&1; echo GT $? >> gpurun_out/q/t.log
python scratch/graph_gap2.py > gpurun_out/q/gg2.log 2>&1
timeout 900 python bench.py --no-cpu > gpurun_out/q/bench_c3.log 2>&1
