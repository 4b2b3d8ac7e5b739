# fused C4 launch time (product library), serial encode/decode split
python tools/profile_c4.py --reps 5 --no-stages 2>&1 | grep "rep [234]"
python tools/profile_c4.py --reps 4 --serial 2>&1 | grep "rep [23]"
