"""Summarise ncu outputs for profiles/ (run here, no GPU needed).

  python tools/ncu_summary.py launches <launches.csv> <out.md>
  python tools/ncu_summary.py full <report.ncu-rep> <out.md> [<traffic.json> <alg_bytes_per_launch>]
"""
import csv, io, json, subprocess, sys, collections


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot = collections.OrderedDict()
    cnt = collections.Counter()
    for r in rows[hdr_i + 1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum":
            continue
        k = r[ik].split("(")[0].replace("void ", "")
        v = float(r[iv].replace(",", ""))
        tot[k] = tot.get(k, 0) + v
        cnt[k] += 1
    unit = "ns"
    s = sum(tot.values())
    lines = [f"# ncu launch list: {path}", "", "`ncu --metrics gpu__time_duration.sum --clock-control none` "
             "(cold-cache, serialised: compare SHARES, not absolutes)", "",
             "| kernel | launches | total ms | share | avg ms |", "|---|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| {k} | {cnt[k]} | {v/1e6:.2f} | {v/s*100:.1f}% | {v/cnt[k]/1e6:.3f} |")
    lines.append(f"| **all** | {sum(cnt.values())} | {s/1e6:.2f} | 100% | |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rep, out, traffic=None, alg=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
            "lts__t_bytes.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"]
    lines = [f"# ncu --set full: {rep}", "", "| metric | value | unit |", "|---|---|---|"]
    for k in want:
        if k in d:
            lines.append(f"| {k} | {d[k]} | {u.get(k, '')} |")
    # stall reasons
    st = {k: v for k, v in d.items() if k.startswith("smsp__average_warp_latency_issue_stalled") or
          k.startswith("smsp__pcsamp_warps_issue_stalled")}
    top = sorted(((k, float(v.replace(",", ""))) for k, v in st.items() if v.replace(",", "").replace(".", "").isdigit()),
                 key=lambda x: -x[1])[:10]
    if top:
        lines += ["", "Top stall-sample counters:", ""] + [f"- {k}: {v:g}" for k, v in top]
    try:
        rd = float(d["dram__bytes_read.sum"].replace(",", ""))
        wr = float(d["dram__bytes_write.sum"].replace(",", ""))
        mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= mul.get(u["dram__bytes_read.sum"], 1)
        wr *= mul.get(u["dram__bytes_write.sum"], 1)
        lines += ["", f"DRAM traffic per launch: {rd + wr:.4g} B (read {rd:.4g}, write {wr:.4g})"]
        if alg:
            lines.append(f"Algorithmic bytes per launch: {float(alg):.4g} B -> traffic/algorithmic = {(rd + wr)/float(alg):.3f}")
        if traffic:
            json.dump({"dram_bytes_per_launch": rd + wr, "read": rd, "write": wr, "source": rep,
                       "alg_bytes_per_launch": float(alg) if alg else None}, open(traffic, "w"), indent=1)
    except Exception as e:
        lines.append(f"(traffic unavailable: {e})")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(*sys.argv[2:])
