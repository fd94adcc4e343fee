set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r2i_pytest_all.log 2>&1; tail -3 gpurun_out/r2i_pytest_all.log
python bench.py > gpurun_out/r2i_bench_5-16.json 2> gpurun_out/r2i_bench_5-16.err; tail -2 gpurun_out/r2i_bench_5-16.err
python bench.py --config 5-8 --no-cpu-baseline > gpurun_out/r2i_bench_5-8.json 2> gpurun_out/r2i_bench_5-8.err
python bench.py --config 5-32 --no-cpu-baseline > gpurun_out/r2i_bench_5-32.json 2> gpurun_out/r2i_bench_5-32.err
python bench.py --config 4 --no-cpu-baseline > gpurun_out/r2i_bench_4.json 2> gpurun_out/r2i_bench_4.err
