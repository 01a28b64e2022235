timeout 900 python -m pytest tests/test_gpu_row.py tests/test_gpu_extra.py tests/test_gpu_parity.py -k "row or c4 or cholesky" -q -s 2>&1 | tail -30 > gpurun_out/r2_row.log
timeout 300 python scratch/rowcg_diag.py > gpurun_out/r2_rowcg_diag.log 2>&1
CURVOPT_PDL=0 timeout 600 python scratch/c4_prof.py > gpurun_out/r2_c4_prof.log 2>&1
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2_bench_c4b.log 2>&1
