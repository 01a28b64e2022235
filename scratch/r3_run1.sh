# fused CG iteration: correctness (GPU suite) + A/B timing
mkdir -p gpurun_out
for f in 0 1; do CURVOPT_CG_FUSED=$f timeout 300 python scratch/phase_time.py > gpurun_out/phase_$f.log 2>&1; done
for f in 0 1; do CURVOPT_CG_FUSED=$f timeout 300 python scratch/cg_fused_check.py > gpurun_out/hash_$f.log 2>&1; done
timeout 300 python bench.py --no-cpu --steps 30 --warmup 5 > gpurun_out/b3f.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gt.log 2>&1; echo GT $? >> gpurun_out/gt.log
