# 1 GPU: final round-end checks
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rs > gpurun_out/r2y_pytest.log 2>&1
tail -4 gpurun_out/r2y_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2y_smoke.log 2>&1
tail -1 gpurun_out/r2y_smoke.log
timeout 900 python bench.py > gpurun_out/r2y_bench_n1.json 2> gpurun_out/r2y_bench_n1.err
timeout 900 python bench.py --impl reference > gpurun_out/r2y_ref_n1.json 2> gpurun_out/r2y_ref_n1.err
