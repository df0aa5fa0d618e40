# 1 GPU: full suite + default bench + A.9 step timeline after the raw-stream change
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rs > gpurun_out/r2s_pytest.log 2>&1
tail -2 gpurun_out/r2s_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2s_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2s_bench_n1.json 2> gpurun_out/r2s_bench_n1.err
timeout 300 python tools/timeline.py gpt2-medium 0.9 a9step > gpurun_out/r2s_timeline_c5_a9step.txt 2>&1
