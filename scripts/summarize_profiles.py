"""Summarise a gpu_round.sh session into profiles/ (tracked): bench lines, the ncu
launch list (per-kernel share of the step), key ncu --set full metrics of the FFN
and router kernels, and FFN per-tile timeline statistics.
Usage: python scripts/summarize_profiles.py <tag>"""
import csv, io, json, os, subprocess, sys

tag = sys.argv[1]
G = "gpurun_out"
P = "profiles"
os.makedirs(P, exist_ok=True)
out = []

def section(t):
    out.append("")
    out.append("## " + t)

for fn in (f"bench_{tag}.json", f"bench_ref_{tag}.json", f"bench_configs_{tag}.json"):
    path = os.path.join(G, fn)
    if os.path.exists(path):
        lines = [l for l in open(path) if l.strip().startswith("{")]
        with open(os.path.join(P, fn.replace(".json", ".jsonl")), "w") as fh:
            fh.writelines(lines)

section("launch list (ncu gpu__time_duration, cold, serialised) — scripts/run_layer.py mixtral 512 3")
path = os.path.join(G, f"launches_{tag}.csv")
if os.path.exists(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    n, v = h.index("Kernel Name"), h.index("Metric Value")
    ours = [(r[n], float(r[v].replace(",", ""))) for r in rows[hi + 1:] if "moe::" in r[n]]
    last = ours[-4:] if len(ours) >= 4 else ours
    tot = sum(t for _, t in last)
    for name, t in last:
        out.append(f"  {t/1e3:9.1f} us  {100*t/tot:5.1f}%  {name[:90]}")
    with open(os.path.join(P, f"launches_{tag}.csv"), "w") as fh:
        fh.write("kernel,ns\n")
        for name, t in ours:
            fh.write(f"\"{name}\",{t:.0f}\n")

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
           "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
           "launch__registers_per_thread", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
traffic = {}
for kern in ("ffn", "router", "router_seg", "dispatch", "combine_token"):
    rep = os.path.join(G, f"prof_{kern}_{tag}.ncu-rep")
    if not os.path.exists(rep):
        continue
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    section(f"ncu --set full: {kern} kernel (Mixtral 512)")
    for row in rows[2:]:
        d = dict(zip(h, row))
        out.append("  kernel: " + d.get("Kernel Name", "")[:100])
        for m in METRICS:
            if m in d:
                out.append(f"  {m:70s} {d[m]:>16s} {units[h.index(m)]}")
        if kern == "ffn":
            try:
                rd = float(d["dram__bytes_read.sum"].replace(",", ""))
                wr = float(d["dram__bytes_write.sum"].replace(",", ""))
                scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
                rd *= scale.get(units[h.index("dram__bytes_read.sum")], 1)
                wr *= scale.get(units[h.index("dram__bytes_write.sum")], 1)
                traffic["mixtral_512_ffn"] = rd + wr
            except Exception:
                pass
if traffic:
    json.dump(traffic, open(os.path.join(P, "traffic.json"), "w"), indent=1)

section("FFN per-tile timelines (scripts/ffn_timeline.py; scripts/timeline_summary.py)")
for c in ("mixtral", "qwen60", "deepseek"):
    if os.path.exists(os.path.join(G, f"timeline_{c}_{tag}.json")):
        r = subprocess.run([sys.executable, "scripts/timeline_summary.py", f"{c}_{tag}"], capture_output=True, text=True)
        out.append("  " + r.stdout.strip())
        os.replace(os.path.join(G, f"timeline_{c}_{tag}.json"), os.path.join(P, f"timeline_{c}_{tag}.json"))

open(os.path.join(P, f"summary_{tag}.md"), "w").write(f"# Profile summary {tag}\n" + "\n".join(out) + "\n")
print("\n".join(out))
