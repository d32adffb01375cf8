#!/bin/bash
# One GPU box pass for a round's evidence: gpu tests, bench lines of every
# config (C4 default with the CPU baseline), the reference arm, the C4 launch
# list and an ncu --set full capture of the hot kernels.
# usage: scripts/round_bench.sh TAG   (outputs gpurun_out/TAG_*)
T=${1:-rX}
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu -rf > $O/${T}_pytest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${T}_smoke.log 2>&1
python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err
for c in C1 C2 C3 C5; do
  python bench.py --config $c --no-cpu --steps 10 > $O/${T}_bench_${c,,}.json 2>> $O/${T}_bench.err
done
python bench.py --impl reference --steps 3 > $O/${T}_bench_reference.json 2>> $O/${T}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${T}_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu > $O/${T}_ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none \
  -k regex:"leg_ana|leg_synth|theta_k2|theta_syn_k2|phi_fwd_k2|phi_inv_k2" -c 16 \
  -o $O/${T}_full python bench.py --steps 1 --warmup 3 --no-cpu > $O/${T}_ncu_full.log 2>&1
# the two-set DMMA analysis launch of the wavelet synthesis (not among the first 16)
ncu --set full --import-source on --clock-control none -k regex:"leg_ana_dmma" -c 2 \
  -o $O/${T}_dmma python bench.py --steps 1 --warmup 3 --no-cpu > $O/${T}_ncu_dmma.log 2>&1
python bench.py --mode shard --no-cpu --steps 10 > $O/${T}_bench_shard1.json 2>> $O/${T}_bench.err
# summaries (text) travel back even when the .ncu-rep files are too large to keep
python scripts/ncu_summary.py full $O/${T}_full.ncu-rep > $O/${T}_full_summary.txt 2>/dev/null
python scripts/ncu_summary.py full $O/${T}_dmma.ncu-rep > $O/${T}_dmma_full_summary.txt 2>/dev/null
# gpurun brings back at most 64 MiB: keep the summaries, drop the reports that do not fit
rm -f $O/${T}_dmma.ncu-rep
[ $(du -sm $O | cut -f1) -gt 60 ] && rm -f $O/${T}_full.ncu-rep
tail -3 $O/${T}_pytest.log; tail -1 $O/${T}_smoke.log
