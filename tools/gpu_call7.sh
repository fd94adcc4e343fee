export HG_CACHE_DIR=/tmp/hgcache_r2
set -x
python tools/prof_stages.py 5-8 2>&1 | grep -v Warn
python bench.py --config 5-8 > gpurun_out/r2_bench_5-8_split.json 2> gpurun_out/r2_bench_5-8_split.err; tail -3 gpurun_out/r2_bench_5-8_split.err
