# Per-op profile of two builds/environments on one box: bash tools/ab_ops.sh "ENV_A" "ENV_B"
A="$1"; B="$2"
env $A timeout 300 python bench.py --no-cpu-baseline --steps 10 --profile-json gpurun_out/ops_A.json > gpurun_out/bA.json 2>/dev/null
env $B timeout 300 python bench.py --no-cpu-baseline --steps 10 --profile-json gpurun_out/ops_B.json > gpurun_out/bB.json 2>/dev/null
python tools/ops_summary.py gpurun_out/ops_B.json gpurun_out/ops_A.json 25
