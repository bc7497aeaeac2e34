import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    print(f.split('/')[-1][:45].ljust(45), 'ms %.3f' % d['ms_per_step'], 'it', d['iterations'],
          {k: (round(v['ms'] * 1e3, 2), v.get('format_frac')) for k, v in d['kernels'].items()})
