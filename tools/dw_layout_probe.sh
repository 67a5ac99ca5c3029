# dW-shaped GEMMs (contraction over tokens) with each operand K-major or MN-major:
# serialized ncu durations after two warm-up launches (tools/gemm_one.py runs 3).
for shape in "768 3072 65536" "768 768 65536"; do
  for ab in "0 0" "1 1" "1 0" "0 1"; do
    echo "== $shape a_kmajor/b_kmajor $ab"
    ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__cycles_elapsed.max \
        --clock-control none -k regex:gemm_tc --launch-skip 2 -c 1 --csv \
        python tools/gemm_one.py $shape $ab 0 0 3 2>/dev/null | grep -E "gpu__time|cycles_elapsed"
  done
done
