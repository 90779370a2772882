"""Aggregate an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel/pass.

usage: launch_summary.py LAUNCHES.csv [BENCH.json]

The launch list covers the first launches of a profiled solve (norm power
iteration first, then a few outer steps), so its raw time shares are not the
solve's.  With a bench line, each pass's cold average over the launches that
did work (duration > NOOP_US; the inner loops enqueue predicted iteration
counts and launches past convergence exit at once) is multiplied by the
solve's real launch count to give a projected share, printed next to the
bench's live (warm, CUDA-event) share."""
import collections
import csv
import json
import re
import sys

NOOP_US = 10.0
KEYS = [("HcgA", "hcg_a"), ("HcgB", "hcg_b"), ("HcgInit", "hcg_init"), ("CgnrInit", "cgnr_init"),
        ("CgnrP1", "cgnr_p1"), ("CgnrP2", "cgnr_p2"), ("CgnrP3", "cgnr_p3"), ("Outer", "outer"),
        ("norm_fused_kernel", "norm_b")]


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == 'ID'][0]
    h = rows[hi]
    ki, mi, vi, ii = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
    per = collections.defaultdict(dict)
    for r in rows[hi + 1:]:
        per[r[ii]][r[mi]] = float(r[vi].replace(',', ''))
        per[r[ii]]['name'] = r[ki]
    return per


def key_of(name):
    m = re.search(r'(?:sweep_kernel|sweep_tma_kernel|sweep_tma2_kernel|pointwise_kernel)<(?:gadi::)?(\w+)<', name)
    return m.group(1) if m else re.sub(r'\(.*', '', name)


def summarize(path, bench=None):
    per = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0, 0.0, 0.0])
    for v in per.values():
        full = v['name']
        a = agg[(key_of(full), full)]
        t = v.get('gpu__time_duration.sum', 0.0)
        d = v.get('dram__bytes_read.sum', 0.0) + v.get('dram__bytes_write.sum', 0.0)
        a[0] += 1
        a[1] += t
        a[2] += d
        if t > NOOP_US * 1e3:
            a[3] += 1
            a[4] += t
            a[5] += d
    tot = sum(a[1] for a in agg.values())
    out = []
    for (k, full), a in sorted(agg.items(), key=lambda x: -x[1][1]):
        na = max(a[3], 1)
        out.append(f"{full[:60]:60s} n={a[0]:5d} active={a[3]:5d} t_active={a[4] / na / 1e3:8.2f}us "
                   f"raw_share={a[1] / tot * 100:5.1f}% dram/active={a[5] / na / 1e6:8.1f}MB "
                   f"dram GB/s={a[5] / max(a[4], 1):6.0f}")
    if bench:
        b = json.load(open(bench))
        ks = b["kernels"]
        proj = {}
        for (k, full), a in agg.items():
            for pat, bk in KEYS:
                if (k == pat or pat in full) and bk in ks and a[3]:
                    # the hot template instance (largest active time) stands for the pass
                    cand = (a[4] / a[3] / 1e3, a[3])
                    if bk not in proj or a[4] > proj[bk][2]:
                        proj[bk] = (cand[0], ks[bk]["active_launches"], a[4])
        ptot = sum(us * n for us, n, _ in proj.values())
        out.append("")
        out.append("projected onto the bench solve (cold ncu avg x real launches) vs bench live share:")
        for bk, (us, n, _) in sorted(proj.items(), key=lambda kv: -kv[1][0] * kv[1][1]):
            out.append(f"  {bk:10s} ncu {us:8.2f}us x {n:5d} -> {us * n / ptot * 100:5.1f}%   "
                       f"live {ks[bk]['avg_us']:8.2f}us, share {ks[bk]['share'] * 100:5.1f}%")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None))
