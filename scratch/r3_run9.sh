mkdir -p gpurun_out/tr
for f in 1 0; do
CURVOPT_CG_FUSED=$f timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu > gpurun_out/tr/tr_$f.log 2>&1
CURVOPT_CG_FUSED=$f timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/tr/plain_$f.log 2>&1
done
