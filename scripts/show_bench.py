"""Print the key fields of a bench.py JSON line (and its sweep)."""
import json
import sys

d = json.load(open(sys.argv[1]))
u = d.get("unfused_baseline") or {}
print(f"value {d['value']:.0f} TF  ms/step {d['ms_per_step']:.3f}  unfused {u.get('value', 0):.0f} TF  "
      f"roofline frac {d['roofline']['frac']:.3f} ({d['roofline']['peak_source']})  "
      f"e2e {d['e2e']['value']:.0f}  clocks {d['clocks']}")
if u.get("interleaved"):
    i = u["interleaved"]
    print(f"interleaved A/B: ours {i['ours_ms_per_step']*1e3:.1f} us  unfused {i['unfused_ms_per_step']*1e3:.1f} us"
          f"  speedup {i['speedup']:.3f}")
b = d["breakdown"]
print(f"ag {b['ag_gemm_ms']*1e3:.0f} us {b['ag_gemm_tflops']:.0f} TF   rs {b['gemm_rs_ms']*1e3:.0f} us "
      f"{b['gemm_rs_tflops']:.0f} TF  tile {b['tile']}")
for s in d.get("sweep") or []:
    print(f"  {s['op']:8s} tp{s['tp']} M={s['M']:6d}  ours {s['ours_us']:7.0f} us {s['ours_tflops_per_gpu']:5.0f} TF"
          f"  unfused {s['unfused_us']:7.0f} us {s['unfused_tflops_per_gpu']:5.0f} TF  frac {s['roofline_frac']:.2f}"
          f"  x{s['unfused_us'] / s['ours_us']:.2f}")
