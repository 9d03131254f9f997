#!/bin/bash
# Regenerate the profiles/ evidence for bench.py's N=1 configuration.
# Run on a GPU box (e.g. under gpurun); each ncu pass runs only after the same
# command has exited 0 without ncu. Outputs go to $1 (default gpurun_out/).
set -e
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
python bench.py --steps 5 --warmup 3 > "$OUT/bench.log" 2>&1
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > "$OUT/bench_short.log" 2>&1
# launch list: per-launch device time of every kernel in 2 timed steps (cold, serialised)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file "$OUT/launches.csv" \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > "$OUT/ncu_launches.log" 2>&1
# one full capture of each attention kernel (4th launch = first timed step)
for k in fa_bwd fa_fwd; do
  ncu --set full --import-source on --clock-control none -k "regex:$k" --launch-skip 3 --launch-count 1 \
      -o "$OUT/${k}_full" -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > "$OUT/ncu_$k.log" 2>&1
  ncu -i "$OUT/${k}_full.ncu-rep" --page details --csv > "$OUT/${k}_details.csv"
  ncu -i "$OUT/${k}_full.ncu-rep" --page raw --csv --metrics \
dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,\
sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,\
l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,\
smsp__issue_active.avg.pct_of_peak_sustained_active > "$OUT/${k}_raw.csv"
done
