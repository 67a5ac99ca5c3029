set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests/test_gpu_multi.py -q --timeout 1500 > gpurun_out/r02_multi4.log 2>&1; echo rc=$? >> gpurun_out/r02_multi4.log
timeout 600 $TR --nproc-per-node 2 --master-port 29611 bench.py --gpus 2 > gpurun_out/r02_bench_n2.json 2> gpurun_out/r02_bench_n2.err
timeout 600 $TR --nproc-per-node 4 --master-port 29612 bench.py --gpus 4 > gpurun_out/r02_bench_n4.json 2> gpurun_out/r02_bench_n4.err
timeout 900 $TR --nproc-per-node 4 --master-port 29613 bench.py --gpus 4 --model 1.3b --tau 8 --batch 32 --micro-batch 16 --clients-per-gpu 2 > gpurun_out/r02_bench_1p3b_n4.json 2> gpurun_out/r02_bench_1p3b_n4.err
timeout 1200 $TR --nproc-per-node 4 --master-port 29614 bench.py --gpus 4 --model 7b --tau 4 --batch 16 --micro-batch 1 --no-agg > gpurun_out/r02_bench_7b_n4.json 2> gpurun_out/r02_bench_7b_n4.err
