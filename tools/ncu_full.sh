#!/bin/bash
# One `ncu --set full` capture of each big kernel of a Random-30 gate pass
# (launches of a gate inside the bench's timed window), after the plain run
# exited 0.  Output: gpurun_out/$1.ncu-rep.   tools/ncu_full.sh LABEL [SKIP]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
LABEL=${1:-full}
SKIP=${2:-1110}   # 4 waves x 6 kernels per gate; gate 46, wave 1
export QCSIM_WAVE_SLICES=256
KERN='regex:^(enc_verify|dec_chunks|enc_lattice|enc_x|tok_emit_codebook|tok_count)'
python bench.py --steps 2 --warmup 3 --parity off --no-accuracy --cpu-budget 1 > gpurun_out/${LABEL}_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/${LABEL}_plain.log; exit 1; }
ncu --set full --clock-control none --import-source on --kernel-name "$KERN" --launch-skip $SKIP --launch-count 6 \
    -o gpurun_out/${LABEL} -f python bench.py --steps 2 --warmup 3 --parity off --no-accuracy --cpu-budget 1 > gpurun_out/${LABEL}_ncu.log 2>&1
echo "ncu=$?"; ls -la gpurun_out/${LABEL}.ncu-rep
