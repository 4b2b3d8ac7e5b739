# A/B of single-signal latencies: HEAD build vs the working tree (GPU side only)
for lib in tools/variants/lib_head.so ""; do
  echo "== lib=${lib:-tree}"
  MSFFT_B200_LIB=$lib python tools/configs_table.py --no-ref ${CONFIGS:-C1 C3 C4 C5} 2>&1 | grep -v SUMMARY | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    if 'gpu_ms' in d: print(d['config'], d['dtype'], d['l'], d['q'], round(d['gpu_ms'],4), {k: round(v,4) for k,v in d.get('gpu_stage_ms',{}).items()})
"
done
