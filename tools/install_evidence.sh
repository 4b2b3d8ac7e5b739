# Copies the judged records of an evidence run (tools/evidence.sh under gpurun)
# from gpurun_out/<tag>/ into profiles/ and profiles/<tag>/.
#   bash tools/install_evidence.sh r02d
set -e
T=${1:?usage: install_evidence.sh <tag>}
O=gpurun_out/$T
P=profiles/$T
test -d "$O"
mkdir -p "$P"
for f in fused_val_ncu_summary fused_val_traffic fused_ncu_summary fused_traffic validate_ncu_summary \
         validate_traffic encode_ncu_summary encode_traffic decode_c4_ncu_summary; do
    cp "$O/$f.json" "profiles/$f.json"
done
cp "$O/c1_decode_ncu_summary.json" "$O/c3_stage_roofline.json" "$O/c5_stage_roofline.json" \
   "$O/c5_run.json" "$O/bench.json" "$O/bench_reference.json" "$O/bench_short.json" \
   "$O/launches_bench.log" "$P/"
python tools/configs_summary.py "$O/configs_table.log" > "$P/configs_table.json"
{
    echo "ncu launch list (gpu__time_duration.sum, --clock-control none) of"
    echo "'python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e', aggregated with tools/ncu_agg.py."
    echo "Per timed validating step: sigma_kernel + fused_val_kernel (scan + encode + decode in one"
    echo "launch); fused_kernel = the ASSUME_VALID steps, validate_kernel = the standalone scan timed"
    echo "for roofline_validate, encode_kernel/decode_kernel = the serial diagnostic pass; the torch"
    echo "kernels generate the synthetic batch, the rest is the plan-time window designer."
    echo
    python tools/ncu_agg.py "$O/launches_bench.csv" 24
} > "$P/launches_summary.txt"
ls "$P"
