set -x
mkdir -p gpurun_out/prof
python bench.py > gpurun_out/prof/bench_full.log 2>&1
python bench.py --impl reference > gpurun_out/prof/bench_ref.log 2>&1
K='regex:^(?!at::|void at::).*'
ncu --profile-from-start off --set full --clock-control none -o /tmp/frame python tools/frame_launches.py > gpurun_out/prof/ncu_frame.log 2>&1
python tools/ncu_summary.py /tmp/frame.ncu-rep gpurun_out/prof/r01_ncu_c2_frame >> gpurun_out/prof/ncu_frame.log 2>&1
ncu --profile-from-start off --set full --clock-control none -o /tmp/train python tools/train_step_once.py > gpurun_out/prof/ncu_train.log 2>&1
python tools/ncu_summary.py /tmp/train.ncu-rep gpurun_out/prof/r01_ncu_c3_train_step >> gpurun_out/prof/ncu_train.log 2>&1
ncu --profile-from-start off --set full --clock-control none -o /tmp/inv python tools/inverse_once.py > gpurun_out/prof/ncu_inv.log 2>&1
python tools/ncu_summary.py /tmp/inv.ncu-rep gpurun_out/prof/r01_ncu_c4_inverse_step >> gpurun_out/prof/ncu_inv.log 2>&1
ls -la gpurun_out/prof
# launch list of the bench command itself (cold, serialised: shares, not values)
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/prof/launches.csv python bench.py --steps 2 --warmup 1 --no-extra --no-cpu-baseline > gpurun_out/prof/ncu_launches.log 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/prof/launches.csv")) if len(r) > 10]
h = rows[0]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}
tot = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    try:
        v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1e-3)
    except ValueError:
        continue
    t = tot[r[ik][:90]]
    t[0] += 1
    t[1] += v
with open("gpurun_out/prof/r01_launch_list_bench.md", "w") as f:
    f.write("| kernel | launches | total us (ncu, serialised) |\n|---|---|---|\n")
    for k, (c, v) in sorted(tot.items(), key=lambda x: -x[1][1]):
        f.write(f"| {k} | {c} | {v:.1f} |\n")
PY
ls -la gpurun_out/prof
