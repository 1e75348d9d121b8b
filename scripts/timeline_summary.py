"""Summarise gpurun_out/timeline_*.json (per-tile FFN timeline)."""
import json, sys
import numpy as np
cfg = {"mixtral": (8, 2, 4096, 14336), "qwen60": (60, 4, 2048, 1408), "deepseek": (256, 8, 7168, 2048), "skew64": (64, 2, 3584, 2560)}
for name in sys.argv[1:] or ["mixtral", "qwen60", "deepseek"]:
    d = json.load(open(f"gpurun_out/timeline_{name}.json"))
    E, k, dd, ff = cfg[name]
    f = np.array(d['fetch_us']); l = np.array(d['load_us']); e = np.array(d['done_us']); sm = np.array(d['sm'])
    n = len(f)
    counts = np.array(d['counts']); bn = 256 if 512 * k > 96 * E else 128
    nch = int(np.sum((counts + bn - 1) // bn)); ngu = nch * ((ff + 127) // 128)
    nsplit = max(1, min(8, (ff + dd // 2) // dd))
    dur = np.zeros(n)
    for s in np.unique(sm):
        ii = np.where(sm == s)[0]; ii = ii[np.argsort(e[ii])]
        prev = 0
        for i in ii:
            dur[i] = e[i] - max(prev, l[i]); prev = e[i]
    gu = np.arange(n) < ngu
    gub = 2 * 128 * dd * 2; dnb = 256 * ff * 2 / nsplit
    last = {s: e[sm == s].max() for s in np.unique(sm)}
    lv = np.array(list(last.values()))
    print(f"{name}: GU {gub/np.median(dur[gu])/1e3:.1f} GB/s/SM | DN {dnb/np.median(dur[~gu])/1e3:.1f} GB/s/SM | "
          f"span {e.max():.1f} us | SM end min/med/max {lv.min():.1f}/{np.median(lv):.1f}/{lv.max():.1f} | "
          f"dep wait mean {np.mean(l[~gu]-f[~gu]):.2f} us")
