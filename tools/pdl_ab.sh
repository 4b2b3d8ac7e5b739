# A/B of the asynchronous bench loop with and without programmatic dependent
# launch (MSFFT_PDL), alternating on one box; device-resident value only.
for i in 1 2 3; do
  for pdl in 0 1; do
    v=$(MSFFT_PDL=$pdl python bench.py --no-cpu --no-e2e --no-clocks 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4))")
    echo "PDL=$pdl $v"
  done
done
