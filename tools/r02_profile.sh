#!/bin/bash
# Round-2 measurement set on one B200 (run under gpurun from the repo root):
# the default bench line, the reference arm, the launch list of the bench
# command, and full ncu captures of the top kernels at C4.
set -u
O=gpurun_out
python bench.py > $O/r02_bench.json 2> $O/r02_bench.err || exit 1
python bench.py --impl reference --steps 2 --warmup 1 > $O/r02_reference.json 2> $O/r02_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file $O/r02_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 --no-traffic > $O/r02_ncu_launch.log 2>&1
REPS=2 ncu --set full --clock-control none --import-source on -k regex:"k_solve_iter" --launch-skip 12 \
    --launch-count 1 -o $O/r02_c4_solve python tools/build_reps.py C4 > $O/r02_ncu_solve.log 2>&1
REPS=2 ncu --set full --clock-control none --import-source on \
    -k regex:"k_aggregate|k_assign_cells|k_pack_members|k_fill_perm" --launch-skip 5 --launch-count 6 \
    -o $O/r02_c4_build python tools/build_reps.py C4 > $O/r02_ncu_build.log 2>&1
ncu --set full --clock-control none -k regex:"k_trace_capture" --launch-count 1 \
    -o $O/r02_c4_trace python tools/trace_times.py C4 > $O/r02_ncu_trace.log 2>&1
ls -la $O
