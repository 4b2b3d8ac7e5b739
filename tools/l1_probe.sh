# fused C4 launch counters with the default carve-out and with 42 KB of extra shared memory
M=gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_op_read_hit_rate.pct,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum,lts__t_sectors_srcunit_tex_op_write.sum
for pad in 0 43008; do
  MSFFT_FUSED_SMEM_PAD=$pad ncu --clock-control none -k regex:fused_kernel -s 1 -c 1 --metrics $M --csv python tools/profile_c4.py --reps 2 --no-stages > gpurun_out/l1_pad$pad.csv 2> gpurun_out/l1_pad$pad.err
done
