import json, glob
for f in sorted(glob.glob('gpurun_out/ab_*.json')):
    try:
        d = json.loads(open(f).read())
        print(f, round(d['ms_per_step'], 2))
    except Exception as e:
        print(f, e)
