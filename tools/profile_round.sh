# Evidence for profiles/<round>/ (run on the GPU box):  bash tools/profile_round.sh round2
R=${1:-round2}; O=gpurun_out/$R; mkdir -p $O
python bench.py --profile-json $O/bench_per_op_profile.json > $O/bench_line.json 2> $O/bench.err
# launch list of the timed step (cold-cache, serialised: use the SHARE of each kernel)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_launches_ncu.csv \
    python bench.py --minimal --steps 2 --warmup 3 > /dev/null 2>&1
# K1 / K5 alone (one launch of each variant), full sections
EB_PROBE_ITERS=1 ncu --set full --import-source on --clock-control none -k regex:"combine|preprocess" \
    -o $O/k1_k5 -f python tools/hbm_kernels_probe.py > /dev/null 2>&1
ncu -i $O/k1_k5.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed > $O/k1_k5_raw.csv 2>/dev/null
# K6 (Track R)
ncu --set full --clock-control none -k regex:"lin1" -c 4 -o $O/k6_lin1 -f python tools/lin1_probe.py 6 3000 > /dev/null 2>&1
ncu -i $O/k6_lin1.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum > $O/k6_lin1_raw.csv 2>/dev/null
# tensor-pipe utilisation / DRAM bytes of every kernel of the timed step (last 2 steps)
ncu --clock-control none --csv --log-file $O/step_kernels_ncu.csv \
    --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed \
    python bench.py --minimal --steps 2 --warmup 3 > /dev/null 2>&1
echo done
