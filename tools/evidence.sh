# Round-2 (final session) evidence on the current code, under gpurun.  Each
# ncu pass runs only after the same command exited 0 alone.  Outputs land in
# gpurun_out/r02d/; the summaries bench.py reads are written there too (copy
# them to profiles/ after checking).
set -x
O=${EVIDENCE_OUT:-gpurun_out/r02d}; mkdir -p $O
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active"
W="C4: 1024 x N=2^22, K=64, complex64 (tools/profile_c4.py)"
# C4 batch: fused, validation scan, serial encode/decode (ncu --set full)
python tools/profile_c4.py --reps 2 --no-stages > $O/profile_c4_plain.log 2>&1 || exit 1
python tools/profile_c4.py --reps 2 --no-stages --serial > $O/profile_c4_serial.log 2>&1 || exit 1
python tools/profile_c4.py --reps 3 --no-stages --validate > $O/profile_c4_validate.log 2>&1 || exit 1
# rep 0 validates (fused_val_kernel), reps 1.. are ASSUME_VALID (fused_kernel)
ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 1 -c 1 \
    -o $O/fused -f python tools/profile_c4.py --reps 3 --no-stages > $O/fused_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused_val_kernel -s 1 -c 1 \
    -o $O/fused_val -f python tools/profile_c4.py --reps 3 --no-stages --validate > $O/fused_val_full.log 2>&1
MSFFT_VAL_FUSED=0 ncu --set full --clock-control none --import-source on -k regex:validate_kernel -c 1 \
    -o $O/validate -f python tools/profile_c4.py --reps 2 --no-stages > $O/validate_full.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:encode_kernel|decode_kernel" -s 2 -c 2 \
    -o $O/serial -f python tools/profile_c4.py --reps 2 --no-stages --serial > $O/serial_full.log 2>&1
python tools/ncu_summary.py $O/fused.ncu-rep --workload "$W" --traffic $O/fused_traffic.json --batch 1024 --n 4194304 > $O/fused_ncu_summary.json
python tools/ncu_summary.py $O/fused_val.ncu-rep --workload "$W, validating" --traffic $O/fused_val_traffic.json --batch 1024 --n 4194304 > $O/fused_val_ncu_summary.json
python tools/ncu_summary.py $O/validate.ncu-rep --workload "$W" --traffic $O/validate_traffic.json --batch 1024 --n 4194304 > $O/validate_ncu_summary.json
python tools/ncu_summary.py $O/serial.ncu-rep --kernel encode_kernel --workload "$W, serial diagnostic" --traffic $O/encode_traffic.json --batch 1024 --n 4194304 > $O/encode_ncu_summary.json
python tools/ncu_summary.py $O/serial.ncu-rep --kernel decode_kernel --workload "$W, serial diagnostic" > $O/decode_c4_ncu_summary.json
# bench launch list (short run), then the bench itself and the reference arm
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/bench_short.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/launches_bench.log 2>&1
# single-signal configs: C1 ncu full of the gated decode, C3/C5 per-stage launch lists
python tools/single_once.py C1 > $O/c1_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k "regex:decode_kernel|encode_kernel" -s 2 -c 2 \
    -o $O/c1 -f python tools/single_once.py C1 > $O/c1_full.log 2>&1
python tools/ncu_summary.py $O/c1.ncu-rep --kernel decode_kernel --workload "C1: N=2^16, K=50, c128 (gated decode)" > $O/c1_decode_ncu_summary.json
python tools/profile_c3.py --reps 2 > $O/c3_plain.log 2>&1 || exit 1
MSFFT_PROFILE_AFTER_PLAN=1 ncu --profile-from-start off --clock-control none --csv --metrics $M \
    python tools/profile_c3.py --reps 2 > $O/c3_stages.csv 2> $O/c3_stages.err
python tools/stage_roofline.py $O/c3_stages.csv --workload "C3: N=2^24, K=1000, c128 (tools/profile_c3.py, serial path)" > $O/c3_stage_roofline.json
python tools/run_c5.py --reps 2 > $O/c5_plain.json 2> $O/c5_plain.err || exit 1
MSFFT_PROFILE_AFTER_PLAN=1 ncu --profile-from-start off --clock-control none --csv --metrics $M \
    python tools/run_c5.py --reps 1 > $O/c5_stages.csv 2> $O/c5_stages.err
python tools/stage_roofline.py $O/c5_stages.csv --anchor-grid-max --workload "C5: N=2^27, K=10^4, c128 (tools/run_c5.py, serial path)" > $O/c5_stage_roofline.json
python tools/run_c5.py --no-stages --reps 5 > $O/c5_run.json 2> $O/c5_run.err
python tools/configs_table.py > $O/configs_table.log 2>&1
# the bench itself on this box, reading the captures above (same native
# sources, so roofline.traffic / pipes are filled), then the reference arm
for f in fused_val_ncu_summary fused_val_traffic fused_ncu_summary fused_traffic validate_ncu_summary \
         validate_traffic encode_ncu_summary encode_traffic decode_c4_ncu_summary; do
    cp $O/$f.json profiles/$f.json
done
python bench.py > $O/bench.json 2> $O/bench.err
python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
ls -la $O
