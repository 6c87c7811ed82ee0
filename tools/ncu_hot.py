"""Developer tool: stall samples by opcode / stall reason and the hottest SASS lines of each kernel in an .ncu-rep."""
import csv, io, subprocess, sys, collections
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(io.StringIO(out)))
kern = []; cur = None
for r in rows:
    if r and r[0] == 'Kernel Name': cur = {'name': r[1], 'hdr': None, 'rows': []}; kern.append(cur); continue
    if cur is None: continue
    if cur['hdr'] is None: cur['hdr'] = r; continue
    cur['rows'].append(r)
seen = set()
for k in kern:
    if k['name'] in seen: continue
    seen.add(k['name'])
    h = k['hdr']; si = h.index('# Samples'); so = h.index('Source'); ie = h.index('Instructions Executed')
    stall_cols = [i for i, c in enumerate(h) if c.startswith('stall_') and 'Not Issued' not in c]
    R = k['rows']; tot = sum(int(r[si]) for r in R); ninst = sum(int(r[ie]) for r in R)
    print("=====", k['name'][:70], "samples", tot, "instructions", ninst)
    byop = collections.Counter(); byn = collections.Counter()
    for r in R:
        t = r[so].split(); op = (t[1] if t[0].startswith('@') else t[0]).split('.')[0]
        byop[op] += int(r[si]); byn[op] += int(r[ie])
    print("  by opcode:", ", ".join(f"{o} {100*c/tot:.1f}% ({byn[o]/1e6:.1f}M)" for o, c in byop.most_common(14)))
    st = collections.Counter()
    for r in R:
        for i in stall_cols: st[h[i]] += int(r[i] or 0)
    print("  stalls:", ", ".join(f"{a[6:]} {100*b/tot:.1f}%" for a, b in st.most_common(9)))
    idx = sorted(range(len(R)), key=lambda i: -int(R[i][si]))[:top]
    for i in sorted(idx):
        r = R[i]; ss = {h[c][6:]: int(r[c] or 0) for c in stall_cols}; m = max(ss, key=ss.get)
        print(f"   {i:5d} {int(r[ie])/1e6:7.2f}M {int(r[si]):6d} {100*int(r[si])/tot:4.1f}% {m:12s} {r[so].strip()[:80]}")
