# time a set of representative conv layers (B=256) through eb_k_conv
for L in "$@"; do echo "$L :: $(timeout 60 python tools/conv_bench.py $L 2>&1 | tail -1)"; done
