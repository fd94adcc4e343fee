export HG_CACHE_DIR=/tmp/hgcache_r2
set -x
python -m pytest tests/test_gpu_large.py -m gpu -x -q -k "5-8" -s > gpurun_out/c5_pytest_58.log 2>&1; tail -12 gpurun_out/c5_pytest_58.log
python tools/prof_stages.py 5-8 > gpurun_out/c5_stages_p2.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches_58_p2.csv python tools/prof_stages.py 5-8 > /dev/null 2>&1
HG_LOCAL_SPLIT=4 python tools/prof_stages.py 5-8 > gpurun_out/c5_stages_p4.log 2>&1 &&
HG_LOCAL_SPLIT=4 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches_58_p4.csv python tools/prof_stages.py 5-8 > /dev/null 2>&1
cat gpurun_out/c5_stages_p2.log gpurun_out/c5_stages_p4.log | grep -v Warn
python -m pytest tests -m gpu -x -q > gpurun_out/c5_pytest_all.log 2>&1; tail -5 gpurun_out/c5_pytest_all.log
