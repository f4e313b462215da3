# Soak of the 8-node layouts on one GPU (the setting of the round-1
# non-finite-logit report): N rounds of 4P_4D and 2P_6D, PD (x=0) and PPD
# (x=1), 6-8 qps, Llama-3-8B shape, device clock. Every run's engine checks
# each sampled id (a non-finite logit row argmaxes to 0x7fffffff and fails the
# run naming node / row / step; PPD_DUMP_BAD_STEP keeps the batch). Summary
# (runs, errors, reductions) in gpurun_out/layouts_soak.json.
#   gpurun --timeout 3600 -- 'bash tools/layouts_soak.sh 12'
N=${1:-10}
O=gpurun_out
: > $O/layouts_soak.log
for i in $(seq 1 $N); do
  qps=$((6 + i % 3))
  PPD_DUMP_BAD_STEP=$O/bad_step_$i.json PPD_LAYOUT_QPS=$qps PPD_LAYOUT_DUR=3 PPD_LAYOUT_KV=2200 \
    PPD_LAYOUTS=4P_4D,2P_6D timeout 600 python tools/layouts_1gpu.py >> $O/layouts_soak.log 2>&1
  echo "round $i qps $qps rc=$?" >> $O/layouts_soak.log
done
python3 - <<'EOF'
import json
runs, errors, red = 0, [], []
for line in open("gpurun_out/layouts_soak.log"):
    line = line.strip()
    if not line.startswith("{"):
        continue
    try:
        d = json.loads(line)
    except ValueError:
        continue
    if "error" in d:
        errors.append(d)
        runs += 1
        continue
    for x in ("x0", "x1"):
        if x in d:
            runs += 1
    if "ttft_t2_p50_reduction" in d:
        red.append(d["ttft_t2_p50_reduction"])
json.dump({"engine_runs": runs, "errors": errors, "ttft_t2_p50_reductions": red}, open("gpurun_out/layouts_soak.json", "w"), indent=1)
print(json.dumps({"engine_runs": runs, "n_errors": len(errors), "reductions": red}))
EOF
