"""One-line-per-config summary of bench JSON lines (development aid)."""
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    t = d.get("time_to_tolerance") or {}
    sp = (t.get("second_pass") or {})
    nd = d.get("near_dstar") or {}
    e = d.get("e2e") or {}
    k = d["roofline"]["kernels"]
    print(f"{f}: {d['value']:.1f} steps/s {d['ms_per_step']:.3f} ms step_frac {d['step_roofline']['frac']:.3f} | "
          + " ".join(f"{n} {v['ms']:.3f}ms/{v['frac']:.2f}" for n, v in k.items())
          + f" skqr {d['roofline']['skqr_ms']:.3f} | ttt {t.get('seconds', 0):.2f}s d*={t.get('d_star')} (oracle {t.get('oracle_d_star')}) "
          f"host {t.get('host_solves')}/{t.get('host_solve_s', 0):.2f}s gpu {t.get('gpu_solves')}/{t.get('gpu_solve_s', 0):.2f}s "
          f"2nd {sp.get('seconds', 0):.2f}s rank {sp.get('rank')} | near {nd.get('value', 0):.1f} steps/s {nd.get('ms_per_step', 0):.2f} ms "
          f"frac {nd.get('step_roofline_frac', 0):.3f} skqr {((nd.get('kernels_ms') or {}).get('skqr') or 0):.3f}ms "
          f"({((nd.get('skqr') or {}).get('frac') or 0):.2f}) | e2e {e.get('value', 0):.1f} steps/s {e.get('seconds', 0):.2f}s")
