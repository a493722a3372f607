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
