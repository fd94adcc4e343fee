export HG_CACHE_DIR=/tmp/hgcache_r2
set -x
python tools/prof_r2.py 5-16 3 1 > gpurun_out/r2b_prof_plain3.log 2>&1 &&
ncu --set full --clock-control none --profile-from-start off -k 'regex:k_b0_gemm_multi|k_zt_multi_pk|k_zy_multi_pk|k_b0_gemv|k_creduce_multi' -c 5 -o /tmp/r2b_full python tools/prof_r2.py 5-16 3 1 > gpurun_out/r2b_ncu_full.log 2>&1
ncu -i /tmp/r2b_full.ncu-rep --page raw --csv > gpurun_out/r2b_full_raw.csv 2> gpurun_out/r2b_full_raw.err
python tools/prof_r2.py 5-8 3 1 > gpurun_out/r2b_prof58_plain3.log 2>&1 &&
ncu --set full --clock-control none --profile-from-start off -k 'regex:k_spike|k_sep_solve|k_local_solve|k_local_panel' -c 8 -o /tmp/r2b_full58 python tools/prof_r2.py 5-8 3 1 > gpurun_out/r2b_ncu_full58.log 2>&1
ncu -i /tmp/r2b_full58.ncu-rep --page raw --csv > gpurun_out/r2b_full58_raw.csv 2> gpurun_out/r2b_full58_raw.err
ls -la gpurun_out | tail -8
