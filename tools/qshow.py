import json
for f in ['q_c2', 'q_c3']:
    try:
        d = json.loads(open('gpurun_out/' + f + '.json').read().strip().splitlines()[-1])
        print(f, round(d['ms_per_step'], 2), round(d['roofline']['frac'], 3), d['clocks']['sm_mhz'])
    except Exception as e:
        print(f, e)
