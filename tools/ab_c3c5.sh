# A/B: single-signal wide-decode configs (C3, C5), HEAD build (tools/variants/lib_head.so)
# vs the working tree, alternating
for i in 1 2; do
  echo "== head"; MSFFT_B200_LIB=tools/variants/lib_head.so python tools/profile_c3.py --no-stages --reps 4 2>&1 | grep "rep 3"
  echo "== new";  python tools/profile_c3.py --no-stages --reps 4 2>&1 | grep "rep 3"
done
echo "== head C5"; MSFFT_B200_LIB=tools/variants/lib_head.so python tools/run_c5.py --no-stages --reps 3 2>&1 | grep -o '"device_ms": \[[^]]*\]'
echo "== new C5";  python tools/run_c5.py --no-stages --reps 3 2>&1 | grep -o '"device_ms": \[[^]]*\]'
