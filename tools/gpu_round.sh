# Round evidence in one gpurun call (1 GPU): ncu --set full captures of one
# C2 frame, one captured C3 training step, one C4 InverseGraph iteration and
# the C5 VQ kernels, summarised into profiles/ (tools/ncu_summary.py), plus the
# launch list of the bench command.  Every program runs once without ncu first.
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh r02'
set -x
R=${1:-r02}
mkdir -p gpurun_out/prof
K='regex:^(?!at::|void at::).*'
for p in frame_launches train_graph_once inverse_once vq_once; do
  python tools/$p.py > gpurun_out/prof/plain_$p.log 2>&1 || exit 1
done
ncu --profile-from-start off --set full --import-source on --clock-control none -o /tmp/frame python tools/frame_launches.py > gpurun_out/prof/ncu_frame.log 2>&1
python tools/ncu_summary.py /tmp/frame.ncu-rep gpurun_out/prof/${R}_ncu_c2_frame >> gpurun_out/prof/ncu_frame.log 2>&1
ncu --profile-from-start off --set full --clock-control none -o /tmp/train python tools/train_graph_once.py > gpurun_out/prof/ncu_train.log 2>&1
python tools/ncu_summary.py /tmp/train.ncu-rep gpurun_out/prof/${R}_ncu_c3_train_step >> gpurun_out/prof/ncu_train.log 2>&1
ncu --profile-from-start off --set full --clock-control none -o /tmp/inv python tools/inverse_once.py > gpurun_out/prof/ncu_inv.log 2>&1
python tools/ncu_summary.py /tmp/inv.ncu-rep gpurun_out/prof/${R}_ncu_c4_inverse_step >> gpurun_out/prof/ncu_inv.log 2>&1
ncu --profile-from-start off --set full --clock-control none -o /tmp/vq python tools/vq_once.py > gpurun_out/prof/ncu_vq.log 2>&1
python tools/ncu_summary.py /tmp/vq.ncu-rep gpurun_out/prof/${R}_ncu_c5_vq >> gpurun_out/prof/ncu_vq.log 2>&1
cp /tmp/frame.ncu-rep gpurun_out/prof/${R}_c2_frame.ncu-rep
# launch list of the bench command itself (cold, serialised: shares, not values)
python bench.py --steps 2 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/prof/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/prof/launches.csv python bench.py --steps 2 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/prof/ncu_launches.log 2>&1
python - "$R" <<'PY'
import csv, collections, sys
R = sys.argv[1]
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
with open(f"gpurun_out/prof/{R}_launch_list_bench.md", "w") as f:
    f.write("| kernel | launches | total us (ncu, serialised) |\n|---|---|---|\n")
    for k, (c, v) in sorted(tot.items(), key=lambda x: -x[1][1]):
        f.write(f"| {k} | {c} | {v:.1f} |\n")
PY
ls -la gpurun_out/prof
