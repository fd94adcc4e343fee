set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r2c_pytest_all.log 2>&1; tail -4 gpurun_out/r2c_pytest_all.log
python bench.py --config 4 > gpurun_out/r2c_bench_4.json 2> gpurun_out/r2c_bench_4.err; tail -2 gpurun_out/r2c_bench_4.err
python bench.py > gpurun_out/r2c_bench_5-16.json 2> gpurun_out/r2c_bench_5-16.err; tail -2 gpurun_out/r2c_bench_5-16.err
