#!/bin/bash
# Round-2 ncu evidence (final code: cut-head backward with early stage release and one dS buffer, head dW from a transposed operand; 3 attention launches
# per layer) for one 125M client step (B=32, S=2048), run on the GPU
# box from the repo root after `python tools/profile_step.py 32` exits 0.
# profile_step runs two rounds of one step each; everything below skips the
# first (warm-up) round's launches.
#   1. launch list of the step (serialised per-launch device times)
#   2. ALL 195 tcgen05 GEMM launches of the second step: time, DRAM bytes,
#      tensor-pipe utilisation (the roofline `traffic` and the per-class table)
#   3. the step's attention launches: tensor pipe, XU (MUFU) and FMA pipes
set -e
mkdir -p gpurun_out/r02d
python tools/profile_step.py 32 > gpurun_out/r02d/r02_profile_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02d/r02_step_launches.csv python tools/profile_step.py 32 > /dev/null 2>&1
PIPE=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second,sm__throughput.avg.pct_of_peak_sustained_elapsed
ncu --metrics $PIPE --clock-control none --csv -k regex:gemm_tc --launch-skip 195 -c 195 \
    --log-file gpurun_out/r02d/r02_gemm_step.csv python tools/profile_step.py 32 > gpurun_out/r02d/r02_ncu_gemm.log 2>&1
ATT=$PIPE,sm__inst_executed_pipe_xu.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tc.sum
ncu --metrics $ATT --clock-control none --csv -k regex:"attn_" --launch-skip 36 -c 36 \
    --log-file gpurun_out/r02d/r02_attn_step.csv python tools/profile_step.py 32 > gpurun_out/r02d/r02_ncu_attn.log 2>&1
ncu --metrics $PIPE --clock-control none --csv -k regex:"ln_|ce_pipe|adamw|colsum|colreduce|embed|splitk|transpose|sum_scaled|aggregate|f32_to" \
    --log-file gpurun_out/r02d/r02_other_step.csv python tools/profile_step.py 32 > gpurun_out/r02d/r02_ncu_other.log 2>&1
echo done
