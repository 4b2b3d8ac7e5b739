# A/B (HEAD build vs working tree) of single-signal latencies and the fused C4 launch
for lib in tools/variants/lib_head.so ""; do
  echo "== lib=${lib:-tree}"
  MSFFT_B200_LIB=$lib python tools/configs_table.py --no-ref C1 C2 C4 2>&1 | grep -v SUMMARY | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    if 'gpu_ms' in d: print(d['config'], d['l'], d['q'], round(d['gpu_ms'],4))
"
  MSFFT_B200_LIB=$lib python tools/profile_c4.py --reps 5 --no-stages 2>&1 | grep "rep [34]"
done
