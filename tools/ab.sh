# A/B: fused C4 launch, HEAD build (tools/variants/lib_head.so) vs the working tree, alternating
for i in 1 2 3; do
  echo "== head"; MSFFT_B200_LIB=tools/variants/lib_head.so python tools/profile_c4.py --reps 5 --no-stages 2>&1 | grep "rep [34]"
  echo "== new";  python tools/profile_c4.py --reps 5 --no-stages 2>&1 | grep "rep [34]"
done
