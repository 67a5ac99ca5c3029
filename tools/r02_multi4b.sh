# 4-GPU check of the current code: the multi-GPU tests (both boundary paths,
# K=8, dropouts) and the N=2 / N=4 125M bench lines
set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests/test_gpu_multi.py -q --timeout 1500 > gpurun_out/m4_multi.log 2>&1; echo rc=$? >> gpurun_out/m4_multi.log
timeout 600 $TR --nproc-per-node 2 --master-port 29611 bench.py --gpus 2 --no-cpu > gpurun_out/m4_bench_n2.json 2> gpurun_out/m4_bench_n2.err
timeout 600 $TR --nproc-per-node 4 --master-port 29612 bench.py --gpus 4 --no-cpu > gpurun_out/m4_bench_n4.json 2> gpurun_out/m4_bench_n4.err
