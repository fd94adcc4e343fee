export HG_CACHE_DIR=/tmp/hgcache_r2
set -x
python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity.py tests/test_gpu_robust.py tests/test_gpu_split.py -m gpu -x -q > gpurun_out/c10_pytest.log 2>&1; tail -3 gpurun_out/c10_pytest.log
python tools/prof_stages.py 5-16 2>&1 | grep -v Warn
HG_Z_PACKED=0 python tools/prof_stages.py 5-16 2>&1 | grep -v Warn
python tools/prof_stages.py 5-32 2>&1 | grep -v Warn
python tools/prof_stages.py 4 2>&1 | grep -v Warn
