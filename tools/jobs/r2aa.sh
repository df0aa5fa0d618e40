# 2 GPUs: NVLink bulk push throughput by op size
mkdir -p gpurun_out
timeout 300 ./tools/nvlink_probe > gpurun_out/r2aa_nvlink_probe.log 2>&1
grep -E "bulk push|remote WRITE" gpurun_out/r2aa_nvlink_probe.log
