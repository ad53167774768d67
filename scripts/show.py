import json, sys, glob
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().split('\n')[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    print(f, '%.3e' % d['value'], round(d['ms_per_step'], 2), {k: round(v, 2) for k, v in d['phase_ms'].items()},
          'surv', d['config'].get('survivors_rank0'), 'frac', round(d['roofline']['frac'], 3))
