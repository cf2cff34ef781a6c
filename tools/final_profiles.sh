#!/bin/bash
# Round evidence for profiles/: one Random-30 gate pass (gate 48, inside the
# bench's timed window) under ncu -- (a) the launch list with duration + DRAM
# bytes of every kernel of the pass, (b) one `--set full` capture of each big
# kernel.  Run only after the plain command exited 0.  tools/final_profiles.sh LABEL
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=${1:-r02}
python tools/prof_run.py random30 1 3 > gpurun_out/${L}_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/${L}_plain.log; exit 1; }
tail -1 gpurun_out/${L}_plain.log
PROF_RANGE=1 ncu --profile-from-start off --clock-control none --csv --log-file gpurun_out/${L}_pass.csv \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed \
    python tools/prof_run.py random30 1 3 > gpurun_out/${L}_pass_ncu.log 2>&1
echo "pass=$?"
PROF_RANGE=1 ncu --profile-from-start off --set full --clock-control none --import-source on \
    --kernel-name 'regex:^(enc_verify|dec_chunks|enc_gate_lattice|tok_emit_codebook|tok_count|enc_chain)$' --launch-count 6 \
    -o gpurun_out/${L}_full -f python tools/prof_run.py random30 1 3 > gpurun_out/${L}_full_ncu.log 2>&1
echo "full=$?"; ls -la gpurun_out/${L}_full.ncu-rep gpurun_out/${L}_pass.csv
