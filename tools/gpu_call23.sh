export HG_CACHE_DIR=/tmp/hgcache_r2f
set -x
python -m pytest tests/test_gpu_multi.py -m gpu -x -q 2>&1 | tail -2
python tools/prof_stages.py 5-16 2>&1 | grep -v Warn
python tools/prof_stages.py 5-8 2>&1 | grep -v Warn
