run() { # up down table tag
python - <<PY > gpurun_out/armvar/$4.json 2> gpurun_out/armvar/$4.err
import sys, runpy
sys.argv = ["bench.py"]
import paper_2601_11822_b200.arm as a
a.MeasuredArm.UP_P99 = $1; a.MeasuredArm.DOWN_P99 = $2; a.MeasuredArm.DOWN_TABLE = $3
runpy.run_path("bench.py", run_name="__main__")
PY
}
mkdir -p gpurun_out/armvar
for r in 1 2; do
run 0.8 0.6 0.7 base_$r
run 0.85 0.65 0.75 m85_$r
run 0.9 0.7 0.8 m90_$r
done
