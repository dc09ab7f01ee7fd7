"""Print the pp kernel's one-round timeline (SVN_PROF=1 run; see kProfTimeline in fused.cuh)."""
import sys
line = [l for l in open(sys.argv[1]) if 'svn prof' in l][-1]
v = [int(x) for x in line.split(']')[1].split()][16:64]
t0 = min(x for x in v if x)
rows = []
for l in range(4):
    for s in range(2):
        i = (l * 2 + s) * 3
        m = [x - t0 if x else None for x in v[i:i + 3]]
        e = [x - t0 if x else None for x in v[24 + i:24 + i + 3]]
        rows.append((l, s, m, e))
print("l s | MMA: wait_start ready committed | EPI: woke worked arrived")
for l, s, m, e in rows:
    print(f"{l} {s} | {m[0]!s:>7} {m[1]!s:>7} {m[2]!s:>7} | {e[0]!s:>7} {e[1]!s:>7} {e[2]!s:>7}")
w = [int(x) for x in line.split(']')[1].split()][16 + 48:16 + 64]
if any(w):
    b = min(x for x in w if x)
    print("last-layer chunks (slot: [start,end] per q):", [[x - b for x in w[s * 8:(s + 1) * 8]] for s in range(2)])
