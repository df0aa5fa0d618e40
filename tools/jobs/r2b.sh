# bulk-copy prune_bitmap / unpack + spec_drop_all: parity, bench A/B, profiles
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu -rs > gpurun_out/r2b_pytest.log 2>&1
tail -3 gpurun_out/r2b_pytest.log
timeout 900 python bench.py > gpurun_out/r2b_bench_c5_n1.json 2> gpurun_out/r2b_bench_c5_n1.err
PACT_BITMAP_CPASYNC=1 PACT_UNPACK_STG=1 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2b_bench_c5_old_n1.json 2> gpurun_out/r2b_bench_c5_old_n1.err
timeout 600 python bench.py --prune per-layer --no-cpu-baseline --no-e2e > gpurun_out/r2b_bench_c5pl_n1.json 2> gpurun_out/r2b_bench_c5pl_n1.err
for C in c1 c2 c3; do
timeout 600 python bench.py --config $C --no-cpu-baseline > gpurun_out/r2b_bench_${C}_n1.json 2> gpurun_out/r2b_bench_${C}_n1.err
PACT_UNPACK_STG=1 timeout 600 python bench.py --config $C --no-cpu-baseline --no-e2e > gpurun_out/r2b_bench_${C}_stg_n1.json 2> gpurun_out/r2b_bench_${C}_stg_n1.err
done
# launch list (cold, serialised) of the default C5 step
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2b_launches_c5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2b_ncu_launch.log 2>&1
# full captures of the hot kernels (the 6th launch of each, warm)
for K in prune_bitmap unpack_kernel pack_lm digest_low; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K --launch-skip 5 -c 1 -o gpurun_out/r2b_full_c5_$K python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2b_ncu_full_$K.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:unpack_kernel --launch-skip 5 -c 1 -o gpurun_out/r2b_full_c2_unpack_kernel python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2b_ncu_full_c2_unpack.log 2>&1
ls -la gpurun_out | tail -30
