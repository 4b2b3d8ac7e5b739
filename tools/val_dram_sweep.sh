mkdir -p gpurun_out/s3
for v in "MSFFT_VAL_CHUNK_MB=32 MSFFT_VAL_EOFF=2 MSFFT_VAL_POLICY=2" "MSFFT_VAL_CHUNK_MB=32 MSFFT_VAL_EOFF=3 MSFFT_VAL_POLICY=2" "MSFFT_VAL_CHUNK_MB=32 MSFFT_VAL_EOFF=1 MSFFT_VAL_POLICY=2" "MSFFT_VAL_CHUNK_MB=16 MSFFT_VAL_EOFF=2 MSFFT_VAL_POLICY=2 MSFFT_VAL_ITEM_KB=64" "MSFFT_VAL_EOFF=-4 MSFFT_VAL_POLICY=7 MSFFT_VAL_ITEM_KB=512"; do
  echo "== $v"
  REPS=3 python tools/val_sweep.py "$v" 2>&1 | tail -1
  REPS=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:fused_val -c 1 python tools/val_sweep.py "$v" 2>&1 | grep -E "dram__|lts__|duration"
done
