#!/bin/bash
# brief bench summary (used during development)
python "$(dirname "$0")/../bench.py" "$@" 2>&1 | tail -1 | python -c "
import json,sys
r=json.loads(sys.stdin.read())
print('value', round(r['value'],2), 'e2e', round(r['e2e']['value'],2), 'err', r['rt_rel_err'])
print({k:round(v['ms_per_step'],3) for k,v in r['stages'].items()})
print('roofline', r['roofline']['kernel'], round(r['roofline']['achieved'],2), round(r['roofline']['frac'],3), 'clk', r['clocks'])"
