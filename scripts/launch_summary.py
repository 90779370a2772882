"""Aggregate an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel/pass."""
import collections, csv, re, sys

def summarize(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == 'ID'][0]
    h = rows[hi]
    ki, mi, vi, ii = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
    per = collections.defaultdict(dict)
    for r in rows[hi + 1:]:
        per[r[ii]][r[mi]] = float(r[vi].replace(',', ''))
        per[r[ii]]['name'] = r[ki]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for v in per.values():
        name = v['name']
        m = re.search(r'(?:sweep_kernel|pointwise_kernel)<gadi::(\w+)<', name)
        key = m.group(1) if m else re.sub(r'\(.*', '', name)
        a = agg[key]
        a[0] += 1
        a[1] += v.get('gpu__time_duration.sum', 0.0)
        a[2] += v.get('dram__bytes_read.sum', 0.0) + v.get('dram__bytes_write.sum', 0.0)
    tot = sum(a[1] for a in agg.values())
    out = []
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:28s} n={a[0]:6d} t_avg={a[1] / a[0] / 1e3:9.2f}us share={a[1] / tot * 100:5.1f}% "
                   f"dram/launch={a[2] / a[0] / 1e6:9.2f}MB  dram GB/s={a[2] / max(a[1], 1):7.0f}")
    return "\n".join(out)

if __name__ == "__main__":
    print(summarize(sys.argv[1]))
