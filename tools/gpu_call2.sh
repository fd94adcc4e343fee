export HG_CACHE_DIR=/tmp/hgcache_r2
set -x
python tools/prof_r2.py 5-16 40 2 > gpurun_out/r2_prof_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2_launches_block_5-16_40it.csv python tools/prof_r2.py 5-16 40 2 > gpurun_out/r2_ncu_launch.log 2>&1
python tools/prof_r2.py 5-16 3 1 > gpurun_out/r2_prof_plain3.log 2>&1 &&
ncu --set full --clock-control none --profile-from-start off -k 'regex:k_local_panel|k_b0_gemm_multi|k_zt_multi|k_zy_multi|k_dots2_batch|k_dcgs2_update|k_assemble_multi|k_spmm|k_local_solve|k_b0_cluster|k_zt$|k_zy$' -c 30 -o /tmp/r2_full python tools/prof_r2.py 5-16 3 1 > gpurun_out/r2_ncu_full.log 2>&1
ncu -i /tmp/r2_full.ncu-rep --page raw --csv > gpurun_out/r2_full_raw.csv 2> gpurun_out/r2_full_raw.err
ncu --set full --clock-control none --import-source on --profile-from-start off -k 'regex:k_local_panel' -c 1 -o /tmp/r2_panel python tools/prof_r2.py 5-16 3 1 > gpurun_out/r2_ncu_panel.log 2>&1
ncu -i /tmp/r2_panel.ncu-rep --page source --csv > gpurun_out/r2_panel_source.csv 2> gpurun_out/r2_panel_source.err
ls -la /tmp/*.ncu-rep
python bench.py --config 5-8 > gpurun_out/r2_bench_5-8.json 2> gpurun_out/r2_bench_5-8.err
python bench.py --config 4 > gpurun_out/r2_bench_4.json 2> gpurun_out/r2_bench_4.err
python tools/prof_multi.py 5-8 16 200 > gpurun_out/r2_prof_multi_5-8.log 2>&1
gzip -f gpurun_out/r2_panel_source.csv
ls -la gpurun_out
