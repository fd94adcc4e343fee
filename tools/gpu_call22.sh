export HG_CACHE_DIR=/tmp/hgcache_r2f
set -x
python tools/prof_r2.py 5-16 40 2 > gpurun_out/r2f_prof_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2f_launches_block_5-16_40it.csv python tools/prof_r2.py 5-16 40 2 > gpurun_out/r2f_ncu_launch.log 2>&1
tail -2 gpurun_out/r2f_ncu_launch.log
