import re, sys, collections
pat = re.compile(r"cta\((\d+),(\d+)\) tid (\d+) bar@(\d+) parity (\d+)(?: raw=(\w+))? prog tma=(-?\d+) mma=(-?\d+) s0=(-?\d+) s1=(-?\d+)")
groups = collections.defaultdict(list)
other = []
for line in sys.stdin:
    m = pat.search(line)
    if not m:
        if "Warning" not in line:
            other.append(line.rstrip())
        continue
    cx, cy, tid, bar, par, raw, tma, mma, s0, s1 = m.groups()
    tid = int(tid)
    role = "sm0" if tid < 128 else "sm1" if tid < 256 else "mma" if tid == 256 else "tma"
    groups[(cx, cy)].append((tid // 32, role, bar, par, raw, tma, mma, s0, s1))
for cta, rows in sorted(groups.items()):
    seen = collections.OrderedDict()
    for w, role, bar, par, raw, tma, mma, s0, s1 in rows:
        seen.setdefault((w, role, bar, par, raw), 0)
        seen[(w, role, bar, par, raw)] += 1
    print("cta", cta, "prog tma=%s mma=%s s0=%s s1=%s" % rows[0][5:])
    for k, n in sorted(seen.items()):
        print("   warp %d %s bar@%s parity %s raw=%s  x%d" % (*k, n))
print("\n".join(other[-10:]))
