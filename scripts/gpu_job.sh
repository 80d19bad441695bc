#!/bin/bash
# One parameterised GPU job runner for gpurun:
#   gpurun --timeout T -- bash scripts/gpu_job.sh <out-dir-name> '<cmd1>' '<cmd2>' ...
# Each command runs in order from the repo root; stdout/stderr go to
# gpurun_out/<name>/NN.log and the exit codes to gpurun_out/<name>/status.txt.
set -u
name=$1; shift
O=gpurun_out/$name
mkdir -p "$O"
python -c "import __graft_entry__ as g; g.build()" > "$O/build.log" 2>&1; echo "build=$?" > "$O/status.txt"
i=0
for cmd in "$@"; do
  i=$((i+1))
  f=$(printf "%s/%02d.log" "$O" "$i")
  echo "# $cmd" > "$f"
  bash -c "$cmd" >> "$f" 2>&1
  echo "$i=$? $cmd" >> "$O/status.txt"
done
echo done >> "$O/status.txt"
