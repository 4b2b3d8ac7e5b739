# Round-2 evidence on the current code (run under gpurun; each ncu pass only
# after the same command exited 0 alone).  Outputs land in gpurun_out/r02/.
set -x
O=gpurun_out/r02; mkdir -p $O
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active"
python tools/profile_c4.py --reps 2 --no-stages > $O/profile_c4_plain.log 2>&1 || exit 1
python tools/profile_c4.py --reps 2 --no-stages --serial > $O/profile_c4_serial.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 1 -c 1 \
    -o $O/fused -f python tools/profile_c4.py --reps 2 --no-stages > $O/fused_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:validate_kernel -c 1 \
    -o $O/validate -f python tools/profile_c4.py --reps 2 --no-stages > $O/validate_full.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:encode_kernel|decode_kernel" -s 2 -c 2 \
    -o $O/serial -f python tools/profile_c4.py --reps 2 --no-stages --serial > $O/serial_full.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/bench_short.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/launches_bench.log 2>&1
python tools/profile_c3.py --reps 2 > $O/c3_plain.log 2>&1 || exit 1
MSFFT_PROFILE_AFTER_PLAN=1 ncu --profile-from-start off --clock-control none --csv --metrics $M \
    python tools/profile_c3.py --reps 2 > $O/c3_stages.csv 2> $O/c3_stages.err
python tools/run_c5.py --reps 2 > $O/c5_plain.json 2> $O/c5_plain.err || exit 1
MSFFT_PROFILE_AFTER_PLAN=1 ncu --profile-from-start off --clock-control none --csv --metrics $M \
    python tools/run_c5.py --reps 1 > $O/c5_stages.csv 2> $O/c5_stages.err
tools/fp64_peak > $O/fp64_peak.log 2>&1
ls -la $O
