timeout 300 python scratch/headdiag2.py scratch/libA.so > gpurun_out/r2_headA2.log 2>&1
timeout 300 python scratch/headdiag2.py scratch/libB.so > gpurun_out/r2_headB2.log 2>&1
