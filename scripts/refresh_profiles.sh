#!/usr/bin/env bash
# Copy the judged evidence of the last gpu_profile.sh call from gpurun_out/ into profiles/<round>/.
set -euo pipefail
R=${1:-r01}
ROOT="$(cd "$(dirname "${BASH_SOURCE[0]}")/.." && pwd)"
O="$ROOT/gpurun_out"; P="$ROOT/profiles/$R"
mkdir -p "$P"
cp "$O/bench.json" "$P/bench.json"
cp "$O/bench_ref.json" "$P/bench_ref.json"
cp "$O/pytest_gpu.log" "$P/pytest_gpu.log"
cp "$O/smoke.log" "$P/smoke.log"
cp "$O/launches.csv" "$P/launches.csv"
python3 "$ROOT/scripts/launch_summary.py" "$O/launches.csv" > "$P/launches_summary.txt"
reps=$(ls "$O"/prof_k_*.ncu-rep)
python3 "$ROOT/scripts/ncu_summary.py" "$P/ncu_summary.json" $reps > "$P/ncu_summary.txt"
cp "$P/ncu_summary.json" "$ROOT/profiles/ncu_summary.json"
for r in $reps; do
  k=$(basename "$r" .ncu-rep); k=${k#prof_}
  python3 "$ROOT/scripts/ncu_hotlines.py" "$r" > "$P/hotlines_$k.txt" || true
done
python3 "$ROOT/scripts/ncu_inst_lines.py" "$O/prof_k_replay.ncu-rep" 60 > "$P/inst_lines_k_replay.txt" || true
python3 "$ROOT/scripts/ncu_inst_lines.py" "$O/prof_k_scan.ncu-rep" 40 > "$P/inst_lines_k_scan.txt" || true
python3 "$ROOT/scripts/sass_mix.py" "$P/k_scan_mix.json" > /dev/null
python3 "$ROOT/scripts/sass_listing.py" "$R" > /dev/null
echo "refreshed $P"
