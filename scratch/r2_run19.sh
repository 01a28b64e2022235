timeout 300 python scratch/headdiag.py scratch/libA.so > gpurun_out/r2_headA.log 2>&1
timeout 300 python scratch/headdiag.py scratch/libB.so > gpurun_out/r2_headB.log 2>&1
