import json, hashlib, time, sys
sys.path.insert(0, '.')
import paper_2011_05698_b200 as M
d = json.load(open('tests/golden/sfft4_c5_windows.json'))
ok = 0
for w in d['windows']:
    t = time.time()
    ww, taps = M.window(w['n'], w['b'], w['delta'])
    sha = hashlib.sha256(taps.astype('<f8').tobytes()).hexdigest()
    same = ww == w['w'] and sha == w['taps_sha256']
    ok += same
    print(w['b'], ww, w['w'], same, f"{time.time()-t:.2f}s", flush=True)
print("identical", ok, "of", len(d['windows']))
