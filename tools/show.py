"""Print the headline numbers of a cycle's outputs: python tools/show.py TAG"""
import json
import sys

tag = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/{tag}_bench.json"))
    r = d["roofline"]
    print(f"bench {d['value'] / 1e6:.1f} M/s {d['ms_per_step']:.4f} ms  e2e {d['e2e']['value'] / 1e6:.1f} M/s  "
          f"roofline {r['kernel']} {r['frac']:.3f}")
    for k, v in r.get("kernels", {}).items():
        print(f"   {k:16s} {v['avg_launch_ms'] * 1e3:7.1f} us  frac {v['frac']:.3f}  share {v['share_of_step']:.3f}")
except Exception as e:
    print("bench:", e)
for c in (4, 5):
    try:
        d = json.load(open(f"gpurun_out/{tag}_config{c}.json"))
        ks = {k: round(v["frac_hbm"], 3) for k, v in d["kernels"].items()}
        print(f"config{c} {d['ms_per_round']:.2f} ms/round {d['triples_per_s'] / 1e6:.2f} M/s {ks} host {d['host_s']}")
        print("   ", {k: v for k, v in list(d["eager_breakdown_ms"].items())[:8]})
    except Exception as e:
        print(f"config{c}:", e)
