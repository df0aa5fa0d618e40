# 1 GPU: hit-tail graph, parity, C5 bench A/B, timelines, ncu of the default kernels
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "prune or reprune or hit_tail or bitmap or unpack_bulk or max_len" > gpurun_out/r2d_pytest.log 2>&1
tail -3 gpurun_out/r2d_pytest.log
timeout 900 python bench.py > gpurun_out/r2d_bench_c5_n1.json 2> gpurun_out/r2d_bench_c5_n1.err
PACT_HIT_GRAPH=0 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2d_bench_c5_nograph_n1.json 2> gpurun_out/r2d_bench_c5_nograph_n1.err
for C in c1 c2 c3 c4; do
timeout 600 python bench.py --config $C --no-cpu-baseline > gpurun_out/r2d_bench_${C}_n1.json 2> gpurun_out/r2d_bench_${C}_n1.err
done
timeout 600 python bench.py --prune per-layer --no-cpu-baseline --no-e2e > gpurun_out/r2d_bench_c5pl_n1.json 2> gpurun_out/r2d_bench_c5pl_n1.err
timeout 900 python bench.py --impl reference > gpurun_out/r2d_ref_c5_n1.json 2> gpurun_out/r2d_ref_c5_n1.err
for S in step a9 hit; do
timeout 300 python tools/timeline.py gpt2-medium 0.9 $S > gpurun_out/r2d_timeline_$S.txt 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2d_launches_c5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2d_ncu_launch.log 2>&1
for K in unpack_kernel digest_low digest_high digest_affine prune_hit; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K --launch-skip 5 -c 1 -o gpurun_out/r2d_full_c5_$K python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2d_ncu_full_$K.log 2>&1
done
for C in c1 c2; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"unpack_kernel|pack_lm" --launch-skip 10 -c 2 -o gpurun_out/r2d_full_${C} python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2d_ncu_full_$C.log 2>&1
done
