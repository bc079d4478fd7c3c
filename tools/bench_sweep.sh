#!/bin/bash
# Bench variants back to back on one box: tools/bench_sweep.sh OUTDIR "N|args" ...
# (each line of OUTDIR/sweep.jsonl = one bench JSON line + the variant)
out=$1; shift
mkdir -p "$out"
port=29600
for spec in "$@"; do
  n=${spec%%|*}; extra=${spec#*|}
  port=$((port + 1))
  if [ "$n" = "1" ]; then
    python bench.py --no-cpu --steps 2 --warmup 3 $extra > "$out/run.log" 2>&1
  else
    python -m torch.distributed.run --nnodes=1 --nproc-per-node "$n" --master-addr 127.0.0.1 \
      --master-port $port bench.py --gpus "$n" --steps 2 --warmup 3 $extra > "$out/run.log" 2>&1
  fi
  line=$(grep '^{' "$out/run.log" | tail -1)
  if [ -n "$line" ]; then
    echo "{\"variant\": \"N=$n $extra\", \"line\": $line}" >> "$out/sweep.jsonl"
  else
    echo "{\"variant\": \"N=$n $extra\", \"error\": \"$(tail -c 300 "$out/run.log" | tr -d '"\n\\')\"}" >> "$out/sweep.jsonl"
  fi
done
