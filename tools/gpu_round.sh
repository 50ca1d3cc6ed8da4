set -x
python -m pytest -q -x tests -m gpu > gpurun_out/pt.txt 2>&1; tail -1 gpurun_out/pt.txt
ncu --set full --import-source on --clock-control none -k regex:"k_(align|torsion|select)" -c 3 -o gpurun_out/prof_r1p python tools/prof_dock.py --ligands 20000 --reps 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1p.csv python bench.py --steps 2 --warmup 1 --ligands 50000 --no-e2e --no-cpu > /dev/null 2>&1
python bench.py > gpurun_out/bench_r1p.log 2>&1; tail -1 gpurun_out/bench_r1p.log
python tools/latency_bench.py > gpurun_out/latency_r1p.log 2>&1; tail -1 gpurun_out/latency_r1p.log
