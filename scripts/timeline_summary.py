"""Summarise gpurun_out/timeline_<tag>.json (per-tile FFN timeline): streaming
rate during the MMA phase, epilogue durations, MMA idle gaps, tail spread."""
import json, sys
import numpy as np
cfg = {"mixtral": (8, 2, 4096, 14336), "qwen60": (60, 4, 2048, 1408), "deepseek": (256, 8, 7168, 2048),
       "skew64": (64, 2, 3584, 2560)}
for tag in sys.argv[1:] or ["mixtral", "qwen60", "deepseek"]:
    path = f"gpurun_out/timeline_{tag}.json"
    import os
    if not os.path.exists(path):
        path = f"profiles/timeline_{tag}.json"
    d = json.load(open(path))
    name = d["config"]
    E, k, dd, ff = cfg[name]
    f = np.array(d["fetch_us"]); e = np.array(d["done_us"]); es = np.array(d["epi_start_us"])
    ms = np.array(d["mma_start_us"]); sm = np.array(d["sm"])
    n = len(f); counts = np.array(d["counts"]); bn = 256 if 512 * k > 96 * E else 128
    nch = int(np.sum((counts + bn - 1) // bn)); ngu = nch * ((ff + 127) // 128); gu = np.arange(n) < ngu
    gap = []
    for s in np.unique(sm):
        ii = np.where(sm == s)[0]; ii = ii[np.argsort(ms[ii])]
        for a, b in zip(ii[:-1], ii[1:]):
            gap.append(ms[b] - es[a])
    lv = np.array([e[sm == s].max() for s in np.unique(sm)])
    mma = es - ms
    print(f"{tag}: GU mma {np.median(mma[gu]):.1f}us epi {np.median((e-es)[gu]):.2f} | DN mma {np.median(mma[~gu]):.1f}us "
          f"epi {np.median((e-es)[~gu]):.2f} | MMA gap med {np.median(gap):.2f} mean {np.mean(gap):.2f} | "
          f"span {e.max():.0f} SM end min/med {lv.min():.0f}/{np.median(lv):.0f}")
