import json,sys
for f in sys.argv[1:]:
    try:
        l=open(f).read().strip().splitlines()[-1]
        d=json.loads(l); r=d['roofline'] or {}
        print(f.split('/')[-1], d['ms_per_step'], d['value'], 'frac', r.get('frac'), 'GB/s', r.get('achieved'), r.get('kernel_ms_by_kind'), r.get('per_round_gbs'))
    except Exception as e: print(f, 'ERR', open(f).read()[-600:])
