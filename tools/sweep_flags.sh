for L in "256 14 14 256 1024 1 1 1 0 --res" "256 28 28 128 512 1 1 1 0 --res" "256 7 7 512 2048 1 1 1 0 --res" "256 14 14 256 256 3 3 1 1" "256 7 7 512 512 3 3 1 1" "256 14 14 1024 256 1 1 1 0" "256 28 28 512 128 1 1 1 0" "256 56 56 256 128 1 1 1 0" "256 28 28 256 512 1 1 2 0"; do
  line="$L ::"
  for E in "X=1" "EB_PAIR=0" "EB_MCAST=0" "EB_RESB=0"; do
    r=$(env $E timeout 60 python tools/conv_bench.py $L 2>&1 | tail -1 | cut -d' ' -f1)
    line="$line [$E] $r"
  done
  echo "$line"
done
