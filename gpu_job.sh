mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
for cfg in c2 c5; do
python bench.py --steps 30 --warmup 5 --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/bench_${cfg}_v4.json 2> gpurun_out/bench_${cfg}_v4.err; echo rc=$?
done
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'pack_kernel|unpack_kernel' -s 4 -c 4 -o gpurun_out/prof_v4 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; echo rc=$?
