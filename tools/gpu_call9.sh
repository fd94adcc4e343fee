export HG_CACHE_DIR=/tmp/hgcache_r2
set -x
python bench.py --config 5-32 > gpurun_out/r2_bench_5-32.json 2> gpurun_out/r2_bench_5-32.err; tail -2 gpurun_out/r2_bench_5-32.err
python bench.py --steps 3 > gpurun_out/r2_bench_5-16_c.json 2> gpurun_out/r2_bench_5-16_c.err; tail -2 gpurun_out/r2_bench_5-16_c.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_reference_arm.json 2> gpurun_out/r2_bench_reference_arm.err; tail -2 gpurun_out/r2_bench_reference_arm.err
