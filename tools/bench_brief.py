"""One-line digest of bench.py JSON lines: python tools/bench_brief.py <file.json> ..."""
import json
import sys

for p in sys.argv[1:]:
    try:
        line = [l for l in open(p) if l.startswith("{")][-1]
        j = json.loads(line)
    except Exception as e:  # noqa: BLE001
        print(p, "unreadable:", e)
        continue
    rf = j.get("roofline", {}) or {}
    at = rf.get("attention", {}) or {}
    ks = rf.get("kernels", {}) or {}
    ck = j.get("clocks", {}) or {}
    print(f"{p}: {j.get('config', {}).get('workload')} value={j.get('value'):.4g} {j.get('unit')} "
          f"ms/step={j.get('ms_per_step'):.4g} e2e={(j.get('e2e') or {}).get('value', 0):.4g} "
          f"clk={ck.get('sm_mhz')} {ck.get('reasons')}")
    for v in ks if isinstance(ks, list) else [at]:
        if isinstance(v, dict) and v:
            print(f"    {v.get('kernel')}: {v.get('bound')} frac={v.get('frac', 0):.3f} ms={v.get('ms_per_launch', 0):.4g} "
                  f"peak={v.get('peak')} ncu={v.get('ncu')}")
    ph = j.get("phases") or {}
    if ph:
        print("    phases:", {k: round(v, 4) for k, v in ph.items() if isinstance(v, float)})
