"""Print compact bench lines: python scripts/bl.py gpurun_out/bench_X.json"""
import json, sys
for f in sys.argv[1:]:
    for ln in open(f):
        if not ln.strip().startswith("{"): continue
        d = json.loads(ln)
        st = d.get("stages_ms") or {}
        print(f"{d['config']['workload'][:34]:34s} B={d['config'].get('tokens')} {d['ms_per_step']*1e3:8.1f}us val={d['value']:.0f} "
              f"e2e={d.get('e2e',{}).get('value',0):.0f} frac={(d.get('roofline') or {}).get('frac',0):.3f} "
              + " ".join(f"{k}={v*1e3:.1f}" for k, v in st.items()) + f" clk={d.get('clocks',{}).get('sm_mhz')}")
