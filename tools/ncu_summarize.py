"""Summarise ncu CSV output into profiles/ (dev tool).
usage: python tools/ncu_summarize.py <launches.csv> <out_prefix> [full_raw.csv ...]"""
import csv, json, sys, collections

def read_launch_list(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
    hdr = rows[hdr_i]
    per = collections.OrderedDict()
    for r in rows[hdr_i + 1:]:
        d = dict(zip(hdr, r))
        k = int(d['ID'])
        e = per.setdefault(k, {'kernel': d['Kernel Name'], 'grid': d.get('Grid Size', '')})
        v = float(d['Metric Value'].replace(',', ''))
        unit = d['Metric Unit']
        scale = {'ns': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(unit, 1)
        name = d['Metric Name']
        if name == 'gpu__time_duration.sum':
            e['us'] = v * scale
        else:
            e[name] = v * scale
    return list(per.values())

def main():
    launches = read_launch_list(sys.argv[1])
    out = sys.argv[2]
    tot_us = sum(e['us'] for e in launches)
    gem = [e for e in launches if 'grouped_gemm' in e['kernel']]
    g_us = sum(e['us'] for e in gem)
    g_rd = sum(e.get('dram__bytes_read.sum', 0) for e in gem)
    g_wr = sum(e.get('dram__bytes_write.sum', 0) for e in gem)
    lines = ["# ncu launch list, one block step (config 2, S=8192, M=8)", "",
             f"{len(launches)} launches, {tot_us/1e3:.2f} ms serialised device time "
             f"(ncu: cold caches, serialised; compare shares, not absolutes).", "",
             f"* mst_grouped_gemm_kernel: {len(gem)} launches, {g_us/1e3:.2f} ms = {100*g_us/tot_us:.1f}% of the step; "
             f"DRAM read {g_rd/1e9:.2f} GB, write {g_wr/1e9:.2f} GB per step "
             f"({(g_rd+g_wr)/max(1,len(gem))/1e9:.3f} GB per launch)", "",
             "| # | kernel | us | DRAM read MB | DRAM write MB |", "|---|---|---|---|---|"]
    for i, e in enumerate(launches):
        lines.append(f"| {i} | {e['kernel'][:40]} | {e['us']:.1f} | {e.get('dram__bytes_read.sum',0)/1e6:.0f} | {e.get('dram__bytes_write.sum',0)/1e6:.0f} |")
    full = []
    for p in sys.argv[3:]:
        rows = list(csv.reader(open(p)))
        hdr, units = rows[0], rows[1]
        keys = ['gpu__time_duration.sum', 'sm__cycles_elapsed.avg.per_second', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
                'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
                'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed',
                'l1tex__m_xbar2l1tex_read_bytes.sum', 'lts__t_sector_hit_rate.pct',
                'launch__registers_per_thread', 'smsp__warps_active.avg.pct_of_peak_sustained_active']
        for r in rows[2:]:
            full.append({'source': p.split('/')[-1], **{k: f"{r[hdr.index(k)]} {units[hdr.index(k)]}" for k in keys if k in hdr}})
    if full:
        lines += ["", "# ncu --set full captures (per launch)", ""]
        for f in full:
            lines.append("* " + ", ".join(f"{'tensor_pipe_active_pct' if 'pipe_tensor' in k else k.split('.')[0]}: {v}" for k, v in f.items()))
    open(out + '.md', 'w').write("\n".join(lines) + "\n")
    json.dump({"dominant_kernel": {"name": "mst_grouped_gemm_kernel", "launches_per_step": len(gem),
                                    "dram_bytes_per_launch": (g_rd + g_wr) / max(1, len(gem)),
                                    "dram_read_bytes_per_step": g_rd, "dram_write_bytes_per_step": g_wr,
                                    "share_of_step_ncu": g_us / tot_us},
               "full_captures": full}, open(out + '.json', 'w'), indent=1)
    print("\n".join(lines[:8]))

main()
