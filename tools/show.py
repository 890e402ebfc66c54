import json,sys
for f in sys.argv[1:]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    k={a:round(b['ms_per_step'],3) for a,b in d['kernels'].items() if b['ms_per_step']>0}
    print(f, f"{d['value']:.3e} p-steps/s  {d['ms_per_step']:.2f} ms/step  frac={d['roofline']['frac']:.3f} step_frac={d['hbm_roofline_step']['frac_of_measured']:.3f}", k, "e2e", d.get('e2e') and f"{d['e2e']['value']:.3e}", d.get('clocks'))
