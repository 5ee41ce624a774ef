import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    k = d.get('kernels', {})
    print(f.split('/')[-1], round(d['value'], 1), 'ms/step', round(d['ms_per_step'], 1),
          'spmv', round(d['roofline']['achieved'] or 0), 'loop', round(d['pcg_loop']['achieved_gbs'] or 0),
          'step_gbs', round(d['pcg_loop']['step_gbs']), {n: round(v['ms'], 1) for n, v in k.items()},
          'e2e', round(d['e2e']['value'], 1))
