#!/bin/bash
# Round evidence (run on the GPU box): GPU tests, bench line, ncu launch list of one reduced
# bench step, ncu --set full captures of every search kernel of the bench (C2 m = 8..1024),
# of C3 / C4 at m = 16 and 64, and of the C5 stress searches (64 MiB slice).  The reports
# are summarised on the box (tools/ncu_summary.py); only the summaries come back.
set -x
mkdir -p /tmp/hcprof
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1 > gpurun_out/parity.txt
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --steps 1 --warmup 3 --per-m 5 --no-e2e --no-cpu > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --per-m 5 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
cap() {  # name, kernel regex, count, profile_search args...
  local name=$1 rx=$2 cnt=$3; shift 3
  python tools/profile_search.py "$@" --reps 1 > gpurun_out/pf_$name.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"$rx" -c $cnt -f -o /tmp/hcprof/$name \
      python tools/profile_search.py "$@" --reps 1 > gpurun_out/ncu_$name.log 2>&1 && \
  python tools/ncu_summary.py /tmp/hcprof/$name.ncu-rep > gpurun_out/ncu_summary_$name.json 2> gpurun_out/ncu_summary_$name.err
}
cap c2 "stream_kernel|gather_kernel" 8 --config C2 --m 8 16 32 64 128 256 512 1024
cap c3 "stream_kernel|gather_kernel" 2 --config C3 --m 16 64
cap c4 "stream_kernel|gather_kernel" 2 --config C4 --m 16 64
cap c5 "stream_kernel|gather_kernel|scan_kernel" 3 --config C5 --n 67108864 --m 32 256
python tools/ncu_lines.py /tmp/hcprof/c2.ncu-rep 'stream_kernel<(int)6' 40 > gpurun_out/ncu_lines_stream_m16.txt 2>&1
python tools/ncu_lines.py /tmp/hcprof/c2.ncu-rep 'gather_kernel<(int)8' 40 > gpurun_out/ncu_lines_gather_m1024.txt 2>&1
rm -rf /tmp/hcprof
echo done
