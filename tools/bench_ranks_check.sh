# Functional check of bench.py's multi-rank path on a one-GPU box: two
# torchrun ranks share the device (gloo for the barrier / max-over-ranks
# reductions; the data path has no collective, so no kernel waits on another
# rank).  Not a timing run.  Expects exactly one JSON line from rank 0 for
# each arm.
export MSFFT_BENCH_DIST_BACKEND=gloo
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29531 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --batch 256 \
    > gpurun_out/ranks_b200.out 2> gpurun_out/ranks_b200.err
echo "b200 arm rc=$?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29532 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 \
    > gpurun_out/ranks_ref.out 2> gpurun_out/ranks_ref.err
echo "reference arm rc=$?"
for f in gpurun_out/ranks_b200.out gpurun_out/ranks_ref.out; do
  python - "$f" <<'PY'
import json, sys
lines = [l for l in open(sys.argv[1]) if l.startswith("{")]
assert len(lines) == 1, f"{sys.argv[1]}: {len(lines)} JSON lines"
d = json.loads(lines[0])
print(sys.argv[1], "n_gpus", d["n_gpus"], "value", round(d["value"], 1), d.get("impl", "b200"),
      "global_batch", d["config"].get("global_batch"), "e2e", (d.get("e2e") or {}).get("value"))
PY
done
