mkdir -p gpurun_out
# C5 path: wall times (graph route) then a launch list of a 3-lambda path with the host-driven loop
python tools/prof_path.py --config C5 --paths 2 > gpurun_out/prof_C5.log 2>&1; cat gpurun_out/prof_C5.log
KG_HOST_LOOP=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C5_r2.csv python tools/prof_path.py --config C5 --paths 1 --n-lambda 3 > gpurun_out/ncu_C5.log 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/launches_C5_r2.csv | head -40
