import csv, collections, json, sys
def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None; data = []
    for r in rows:
        if r and r[0] == 'ID': hdr = r; continue
        if hdr and len(r) == len(hdr): data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(list)
    for d in data: agg[d['Kernel Name'][:70]].append(float(d['Metric Value']))
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{sum(v)/1e3:9.1f} us  n={len(v):4d}  avg={sum(v)/len(v)/1e3:7.2f} us  {k}")
def bench(path):
    for line in open(path):
        if line.startswith('{'):
            d = json.loads(line)
            print({k: d[k] for k in ('value','graph_renders_per_sec','ms_per_step') if k in d}, 'e2e', d.get('e2e',{}).get('value'), 'cpu', d.get('cpu_baseline',{}).get('value'), d.get('clocks'))
            for t, v in sorted(d.get('roofline_by_step_type', {}).items(), key=lambda kv: -kv[1]['ms']):
                print(f"  {t:10s} {v['ms']*1e3:8.1f} us  {v['achieved_gbs']:8.0f} GB/s  share {v['share']:.2f}")
if __name__ == '__main__':
    (bench if sys.argv[1] == 'bench' else launches)(sys.argv[2])
