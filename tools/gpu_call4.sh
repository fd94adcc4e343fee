export HG_CACHE_DIR=/tmp/hgcache_r2
set -x
python -m pytest tests/test_gpu_split.py -m gpu -x -q > gpurun_out/c4_pytest_split.log 2>&1; tail -15 gpurun_out/c4_pytest_split.log
for sp in auto 1 2 8; do
  HG_LOCAL_SPLIT=$sp python tools/prof_stages.py 5-8
done 2>&1 | grep -v Warning | tee gpurun_out/c4_stages.log
python -m pytest tests -m gpu -x -q > gpurun_out/c4_pytest_all.log 2>&1; tail -5 gpurun_out/c4_pytest_all.log
