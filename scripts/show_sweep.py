import json, sys
for ln in open(sys.argv[1]):
    try:
        d = json.loads(ln)
    except Exception:
        print(ln.rstrip()[:200]); continue
    s = f"{d['config']:28s} K1 {d['k1_ms']:.3f} ms {d['k1_gbs']:.0f} GB/s frac {d['k1_frac']:.3f}"
    if 'k3_ms' in d:
        s += f" | K3 {d['k3_ms']:.3f} ms frac {d['k3_frac']:.3f}"
    if 'gpu_solve' in d:
        g = d['gpu_solve']
        s += f" | solve {g['status']} {g['outer']}/{g['inner']} {g['wall_s']*1e3:.1f} ms ({g.get('ms_per_inner_iteration',0):.3f} ms/it)"
    print(s)
