"""Prints the SUMMARY rows of a tools/configs_table.py log as indented JSON.
usage: python tools/configs_summary.py configs_table.log > configs_table.json"""
import json
import sys

rows = None
for ln in open(sys.argv[1]):
    if ln.startswith("SUMMARY "):
        rows = json.loads(ln[8:])
if rows is None:
    sys.exit("no SUMMARY line in " + sys.argv[1])
json.dump(rows, sys.stdout, indent=1)
print()
