#!/bin/bash
# ncu evidence for one 125M client step (run on the GPU box from the repo root,
# after the same command has exited 0 without ncu).  Summaries land in
# gpurun_out/*.txt|json (the .ncu-rep files are large; kept only if small).
#   1. launch list (serialised, cold-cache per-launch times) of one step
#   2. DRAM bytes of every GEMM launch of one step (roofline traffic)
#   3. --set full of one layer's kernels (GEMM classes, attention, LN, CE)
set -e
mkdir -p gpurun_out
python tools/profile_step.py 32 > gpurun_out/profile_step_plain.log 2>&1
# profile_step runs two rounds of one step; round 1 is the warm-up
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/step_launches.csv python tools/profile_step.py 32 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:gemm_tc --launch-skip 72 -c 72 -o gpurun_out/gemm_dram -f \
    python tools/profile_step.py 32 > gpurun_out/ncu_gemm.log 2>&1
python tools/ncu_summary.py gpurun_out/gemm_dram.ncu-rep gpurun_out/r_gemm_dram
ncu --set full --clock-control none --import-source on -k regex:gemm_tc --launch-skip 72 -c 12 \
    -o gpurun_out/gemm_full -f python tools/profile_step.py 32 > gpurun_out/ncu_gemm_full.log 2>&1
python tools/ncu_summary.py gpurun_out/gemm_full.ncu-rep gpurun_out/r_gemm_full
ncu --set full --clock-control none --import-source on -k regex:"attn_|ln_|ce_pipe|adamw|colsum" \
    --launch-skip 176 -c 16 -o gpurun_out/other_full -f python tools/profile_step.py 32 \
    > gpurun_out/ncu_other_full.log 2>&1
python tools/ncu_summary.py gpurun_out/other_full.ncu-rep gpurun_out/r_other_full
ls -la gpurun_out
# keep the reports only if they fit the 64 MiB copy-back
for f in gpurun_out/*.ncu-rep; do [ $(stat -c %s $f) -lt 20000000 ] || rm -f $f; done
echo done
