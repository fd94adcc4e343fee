export HG_CACHE_DIR=/tmp/hgcache_r2
set -x
python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity.py tests/test_gpu_robust.py -m gpu -x -q > gpurun_out/c3_pytest.log 2>&1; tail -3 gpurun_out/c3_pytest.log
for cfg in 5-8 5-16 4; do
  python tools/prof_stages.py $cfg
  HG_PANEL_CSPLIT=1 python tools/prof_stages.py $cfg
  HG_PANEL_CSPLIT=0 python tools/prof_stages.py $cfg
  HG_B0_DENSE=1 python tools/prof_stages.py $cfg
done 2>&1 | grep -v Warning | tee gpurun_out/c3_stages.log
