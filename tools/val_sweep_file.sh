# runs tools/val_sweep.py over the variants listed one per line in $1
mapfile -t V < "$1"
python tools/val_sweep.py "${V[@]}"
