#!/bin/bash
# per-launch ncu durations of the kernels matching REGEX in one C4 bench step
# (development aid): scripts/ncu_kernel_times.sh REGEX [COUNT] [bench args...]
re=$1; n=${2:-6}; shift; shift
f=$(mktemp)
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$re" -c $n --csv --log-file $f \
  python bench.py --steps 1 --warmup 3 --no-cpu "$@" > /dev/null 2>&1
python - $f <<'PY'
import csv,sys
rows=[r for r in csv.reader(open(sys.argv[1])) if 'Kernel Name' in r or (len(r)>10 and r[0].isdigit())]
hdr=rows[0]; ki=hdr.index('Kernel Name'); vi=hdr.index('Metric Value'); gi=hdr.index('Grid Size')
for r in rows[1:]:
    print(r[ki][:40], r[gi], r[vi])
PY
rm -f $f
