# 1 GPU: the round-end checks on the final tree (full GPU suite, smoke, default bench, reference arm)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rs > gpurun_out/r2k_pytest.log 2>&1
tail -4 gpurun_out/r2k_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2k_smoke.log 2>&1
tail -1 gpurun_out/r2k_smoke.log
timeout 900 python bench.py > gpurun_out/r2k_bench_n1.json 2> gpurun_out/r2k_bench_n1.err
timeout 900 python bench.py --impl reference > gpurun_out/r2k_ref_n1.json 2> gpurun_out/r2k_ref_n1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2k_launches_c5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2k_ncu_launch.log 2>&1
for K in unpack_kernel pack_lm prune_bitmap; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K --launch-skip 5 -c 1 -o gpurun_out/r2k_full_c5_$K python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2k_ncu_full_$K.log 2>&1
done
