# ncu evidence for the C3 bench step: launch list (time + DRAM bytes per launch) of two graph-replayed
# steps, and one --set full capture of the attention kernel at the C3 shape
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/c3_step_launches.csv python scripts/prof_step.py --steps 2 > /dev/null 2>&1
echo launches_rc=$?
ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 3 -c 1 -o gpurun_out/attn_c3 \
    python scripts/attn_perf.py --seqs 16 --new 64 --cached 5120 --dh 128 --reps 2 > /dev/null 2>&1
echo full_rc=$?
ls -la gpurun_out/
