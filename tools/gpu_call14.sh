export HG_CACHE_DIR=/tmp/hgcache_r2
set -x
python tools/prof_stages.py 5-16 2>&1 | grep -v Warn
HG_B0_SPLIT_CS=4 python tools/prof_stages.py 5-16 2>&1 | grep -v Warn
python tools/prof_stages.py 4 2>&1 | grep -v Warn
