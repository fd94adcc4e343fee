export HG_CACHE_DIR=/tmp/hgcache_r2
set -x
python -m pytest tests/test_gpu_b0split.py -m gpu -x -q 2>&1 | tail -15
python tools/prof_stages.py 5-16 2>&1 | grep -v Warn
python tools/prof_stages.py 4 2>&1 | grep -v Warn
