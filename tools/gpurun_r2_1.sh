cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/r2_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/r2_gputest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
tail -3 gpurun_out/r2_gputest.log; cat gpurun_out/r2_bench.json | head -c 3000
