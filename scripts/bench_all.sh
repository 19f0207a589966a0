#!/usr/bin/env bash
# Every bench workload (both arms) on one box -> gpurun_out/<round>/bench_*.json
R=${1:-r02}
O=gpurun_out/$R
mkdir -p $O
for wl in train augment clip train-l14 feed; do
  python bench.py --workload $wl --steps 10 --warmup 3 > $O/bench_$wl.json 2> $O/bench_$wl.err
  python bench.py --impl reference --workload $wl --steps 5 --warmup 3 > $O/bench_ref_$wl.json 2> $O/bench_ref_$wl.err
done
python -m pytest tests -m gpu -q > $O/gputest.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
tail -2 $O/gputest.txt
