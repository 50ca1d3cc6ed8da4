# GPU pass of a round (run under gpurun): tests, smoke, ncu capture + launch list, bench, reference arm.
# Outputs land in gpurun_out/ (scratch); summaries go to profiles/ with tools/ncu_summary.py (run here).
set -x
TAG=${TAG:-r2}
python -m pytest -q -x tests -m gpu > gpurun_out/pt_$TAG.txt 2>&1; tail -1 gpurun_out/pt_$TAG.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1; tail -1 gpurun_out/smoke_$TAG.txt
ncu --set full --import-source on --clock-control none -k regex:"k_(align|torsion|select)" -c 3 -o gpurun_out/prof_$TAG python tools/prof_dock.py --ligands 20000 --reps 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_(align_latency|optimize_latency)" -c 3 -o gpurun_out/prof_lat_$TAG python tools/prof_dock.py --c2 --family latency --reps 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --ligands 50000 --no-e2e --no-cpu --no-extras > /dev/null 2>&1
python bench.py > gpurun_out/bench_$TAG.log 2>&1; tail -1 gpurun_out/bench_$TAG.log | cut -c1-400
python bench.py --impl reference > gpurun_out/benchref_$TAG.log 2>&1; tail -1 gpurun_out/benchref_$TAG.log | cut -c1-300
