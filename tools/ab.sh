# A/B a layer list under two environment settings, interleaved on the same box:
#   bash tools/ab.sh "ENV_A" "ENV_B" "layer args" ["layer args" ...]
A="$1"; B="$2"; shift 2
for L in "$@"; do
  for rep in 1 2; do
    ra=$(env $A timeout 60 python tools/conv_bench.py $L 2>&1 | tail -1 | cut -d' ' -f1)
    rb=$(env $B timeout 60 python tools/conv_bench.py $L 2>&1 | tail -1 | cut -d' ' -f1)
    echo "$L :: [$A] $ra us  [$B] $rb us"
  done
done
