# Round-end evidence on the current code: bench (both arms), the ncu launch
# list of a short bench run, and one `ncu --set full` capture of the fused
# C4 launch.  Each ncu pass runs only after the same command exited 0 alone.
set -x
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err || exit 1
python bench.py --impl reference > gpurun_out/bench_reference_final.json 2> gpurun_out/bench_reference_final.err
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_short.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/launches_final.log 2>&1
python tools/profile_c4.py --reps 2 --no-stages > gpurun_out/profile_c4_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 1 -c 1 \
    -o gpurun_out/fused_final -f python tools/profile_c4.py --reps 2 --no-stages > gpurun_out/fused_full.log 2>&1
