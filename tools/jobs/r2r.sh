# 1 GPU: where the C5 A.9 step's time goes (CUPTI timeline of prune + masked_allreduce)
mkdir -p gpurun_out
timeout 300 python tools/timeline.py gpt2-medium 0.9 a9step > gpurun_out/r2r_timeline_c5_a9step.txt 2>&1
