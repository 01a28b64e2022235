set -x
mkdir -p gpurun_out/r3b
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r3b/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/r3b/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3b/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r3b/bench_c3.log 2>&1
timeout 900 python bench.py --config cadence --steps 300 --warmup 3 > gpurun_out/r3b/bench_cad.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r3b/bench_torchrun1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file /tmp/c3_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1
gzip -c /tmp/c3_launches.csv > gpurun_out/r3b/c3_launches.csv.gz
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_cg_fused -c 12 --csv --log-file gpurun_out/r3b/cg_fused_ncu.csv python scratch/cg_fused_check.py > /dev/null 2>&1
for f in 0 1; do echo "CURVOPT_CG_FUSED=$f"; CURVOPT_CG_FUSED=$f timeout 300 python scratch/cg_iter_time.py; done > gpurun_out/r3b/cg_iter_time.log 2>&1
