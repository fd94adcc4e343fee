set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r2g_pytest_all.log 2>&1; tail -3 gpurun_out/r2g_pytest_all.log
python bench.py > gpurun_out/r2g_bench_5-16.json 2> gpurun_out/r2g_bench_5-16.err; tail -2 gpurun_out/r2g_bench_5-16.err
python bench.py --impl reference > gpurun_out/r2g_bench_ref.json 2> gpurun_out/r2g_bench_ref.err; tail -1 gpurun_out/r2g_bench_ref.json | head -c 600
