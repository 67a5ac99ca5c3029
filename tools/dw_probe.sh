set -x
for g in 1 4 8 16; do PHOTON_GEMM_GROUP=$g python tools/gemm_one.py 768 3072 65536 0 0 0 0 10; done
PHOTON_GEMM_PAIR=0 python tools/gemm_one.py 768 3072 65536 0 0 0 0 10
python tools/gemm_one.py 768 3072 65536 0 0 0 0 10
python tools/gemm_one.py 768 3072 65536 1 1 0 0 10
python tools/gemm_one.py 768 3072 65536 1 0 0 0 10
python tools/gemm_one.py 768 3072 65536 0 1 0 0 10
ncu --set full --clock-control none -k regex:gemm_tc -c 1 -o gpurun_out/dw_mn python tools/gemm_one.py 768 3072 65536 0 0 0 0 1
ncu --set full --clock-control none -k regex:gemm_tc -c 1 -o gpurun_out/dw_km python tools/gemm_one.py 768 3072 65536 1 1 0 0 1
ls -la gpurun_out
