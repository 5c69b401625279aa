"""Print step / stage / kernel-class times of gpurun_out/sw_<name>.json files."""
import json, sys
for n in sys.argv[1:]:
    try:
        d = json.load(open(f"gpurun_out/sw_{n}.json"))
    except Exception as e:
        print(n, "ERR", e); continue
    k = d["roofline"]["kernels"]
    print(n, f"step {d['ms_per_step']:.2f} e2e {d['e2e']['value']/1e6:.1f}M",
          " ".join(f"{a}={v:.2f}" for a, v in d["stage_ms"].items()),
          " ".join(f"{a}={k[a]['avg_ms']:.3f}" for a in k))
