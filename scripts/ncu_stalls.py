"""Top stall sites of the first kernel (or the one matching argv[2]) in an ncu report."""
import csv, subprocess, sys

rep = sys.argv[1]
pat = sys.argv[2] if len(sys.argv) > 2 else None
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
kern, out, cur = None, [], None
for r in rows:
    if r and r[0] == 'Kernel Name':
        cur = r[1]
        continue
    if pat and (cur is None or pat not in cur):
        continue
    if kern is None:
        kern = cur
    if cur != kern:
        break
    if len(r) > 4 and r[0].startswith('0x'):
        out.append((r[0], int(r[2]), r[1].strip(), int(r[5])))
tot = sum(o[1] for o in out)
print(kern[:100], 'samples', tot)
for i, (a, s, src, ex) in enumerate(out):
    if s > 0.04 * tot:
        for j in range(max(0, i - 4), min(len(out), i + 2)):
            print(f"  {out[j][0][-5:]} {out[j][1]:5d} {out[j][3]:8d} {out[j][2]}")
        print('  ----')
