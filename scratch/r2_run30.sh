timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r2_gputest.log
timeout 1200 ncu --profile-from-start off -k "regex:k_(flat|cg|norm|apply|rad|hutch|diag|chain|trace)" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_c5_vec.csv python scratch/c5_step.py > gpurun_out/r2_c5_step.log 2>&1
python scratch/vec_sum.py gpurun_out/r2_c5_vec.csv > gpurun_out/r2_c5_vec_table.txt 2>&1
