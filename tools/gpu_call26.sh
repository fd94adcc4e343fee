export HG_CACHE_DIR=/tmp/hgcache_r2g
set -x
python tools/prof_r2.py 4 3 1 > gpurun_out/r2j_plain.log 2>&1 &&
ncu --set full --clock-control none --profile-from-start off -k 'regex:k_spmm|k_b0s_|k_b0_cluster' -c 10 -o /tmp/r2j_full python tools/prof_r2.py 4 3 1 > gpurun_out/r2j_ncu.log 2>&1
ncu -i /tmp/r2j_full.ncu-rep --page raw --csv > gpurun_out/r2j_full_raw.csv 2> gpurun_out/r2j_full_raw.err
python tools/prof_r2.py 5-16 3 1 > gpurun_out/r2j_plain516.log 2>&1 &&
ncu --set full --clock-control none --profile-from-start off -k 'regex:k_spmm' -c 3 -o /tmp/r2j_spmm python tools/prof_r2.py 5-16 3 1 > gpurun_out/r2j_ncu516.log 2>&1
ncu -i /tmp/r2j_spmm.ncu-rep --page raw --csv > gpurun_out/r2j_spmm_raw.csv 2> /dev/null
ls -la gpurun_out | tail -6
