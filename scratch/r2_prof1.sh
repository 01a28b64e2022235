# Round-2 evidence: product full capture, C3 bench launch list, cadence launch list
bash scratch/capture_product.sh r2 > gpurun_out/r2_capture.log 2>&1
python scratch/product_traffic.py gpurun_out/r2_product_full_raw.csv gpurun_out/r2_product_traffic.json > gpurun_out/r2_product_traffic.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c3_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r2_c3_ncu_bench.log 2>&1
python scratch/launch_sum.py gpurun_out/r2_c3_launches.csv > gpurun_out/r2_c3_launch_sum.txt 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_cad_launches.csv python scratch/cadence_prof.py > /dev/null 2>&1
python scratch/launch_sum.py gpurun_out/r2_cad_launches.csv > gpurun_out/r2_cad_launch_sum.txt 2>&1
