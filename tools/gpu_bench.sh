# bench line + reference arm + ncu launch list + one ncu --set full capture of the top kernel
set -x
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches_wan.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --sp-sim 0 > gpurun_out/${TAG}_ncu_b.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_attn_fwd -s 3 -c 1 -o gpurun_out/${TAG}_wan_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --sp-sim 0 > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
cat gpurun_out/${TAG}_bench.json | head -c 3000
