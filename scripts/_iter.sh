mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "build or hist" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pt.log
for HB in 1 0; do
PCT_HIST_BULK=$HB timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/b3_$HB.log 2>&1; echo "b3 $HB rc=$?"; python - <<PY
import json; d=json.loads(open("gpurun_out/b3_$HB.log").read().strip().splitlines()[-1]); print("HB=$HB", round(d["ms_per_step"],3), {k:round(v,3) for k,v in d.get("stages_ms").items()}, d.get("parity",{}).get("ok"))
PY
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/l3.csv python bench.py --config 3 --profile --no-e2e --no-cpu --no-parity > /dev/null 2>&1; echo "ncu rc=$?"
cp gpurun_out/l3.csv gpurun_out/launches_l3.csv; python scripts/launch_table.py l3 | tail -14
