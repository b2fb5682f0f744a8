#!/bin/bash
# One GPU session: build, smoke, GPU tests, bench, ncu launch list + full captures.
# Usage (from the repo root, under gpurun): bash scripts/gpu_check.sh MODE
# MODE: all | tests | bench | c3 | ncu | quick | prof | diag3 | sign | signprof | clean |
#       probe | kint | mesh | e2e | init | final (TAG=rNN: full capture into gpurun_out/$TAG)
set -u
mkdir -p gpurun_out
what=${1:-all}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
(nproc; free -g) >> gpurun_out/gpu.txt 2>&1
python -m paper_2512_11473_b200.build > gpurun_out/build.log 2>&1
python -c "import oracle.oracle as o; o.build()" >> gpurun_out/build.log 2>&1
if [[ $what == all || $what == tests ]]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
  timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
if [[ $what == all || $what == bench ]]; then
  timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
fi
if [[ $what == all || $what == c3 ]]; then
  timeout 900 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
  timeout 900 python bench.py --config C5 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_sweep|k_reinit|k_gradient|k_kint' -s 26 -c 3 -o gpurun_out/prof_c3 python bench.py --config C3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c3.log 2>&1
fi
if [[ $what == all || $what == ncu ]]; then
  B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_reinit|k_sweep' -s 25 -c 1 -o gpurun_out/prof_reinit $B > gpurun_out/ncu_reinit.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gradient|k_kint|k_probe|k_phi_init|k_count|k_tag|k_nb' -s 7 -c 7 -o gpurun_out/prof_other $B > gpurun_out/ncu_other.log 2>&1
fi
ls -la gpurun_out > gpurun_out/ls.txt
if [[ $what == quick ]]; then
  timeout 300 python -m pytest tests -m gpu -q -x -k "reinit or slab or c3" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
  timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
fi
if [[ $what == prof ]]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_probe|k_kint|k_gradient|k_phi_init|k_nb|k_tag" -s 6 -c 6 -o gpurun_out/prof_b python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1
fi
if [[ $what == diag3 ]]; then
  timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
  SG_TAG_CULL=0 timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_nocull.json 2> gpurun_out/bench_c3_nocull.err
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --config C3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_c3.log 2>&1
fi
if [[ $what == sign ]]; then
  timeout 900 python -m pytest tests/test_sign_gpu.py -q -x -rf > gpurun_out/pytest_sign.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sign.log
  timeout 600 python scripts/sign_bench.py C2 C3 > gpurun_out/sign_bench.json 2> gpurun_out/sign_bench.err
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sign.csv python scripts/sign_bench.py C2 > gpurun_out/ncu_sign.log 2>&1
fi
if [[ $what == signprof ]]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_cell_sweep|k_pt_sweep|k_pt_apply|k_nb_fix|k_bg_fix' -s 120 -c 6 -o gpurun_out/prof_sign python scripts/sign_bench.py C3 > gpurun_out/ncu_signprof.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 700 --log-file gpurun_out/launches_sign_c3.csv python scripts/sign_bench.py C3 > gpurun_out/ncu_sign_c3.log 2>&1
fi
if [[ $what == clean ]]; then
  timeout 900 python -m pytest tests/test_clean_gpu.py tests/test_sign_gpu.py -q -x -rf > gpurun_out/pytest_clean.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_clean.log
  timeout 600 python scripts/clean_bench.py C2 FIN128 > gpurun_out/clean_bench.json 2> gpurun_out/clean_bench.err
fi
if [[ $what == probe ]]; then
  timeout 600 python -m pytest tests -m gpu -q -x -k "probe or smoke or c5 or slab" > gpurun_out/pytest_probe.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_probe.log
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
  timeout 600 python bench.py --no-cpu-baseline --order shuffled > gpurun_out/bench_shuf.json 2> /dev/null
fi
if [[ $what == kint ]]; then
  timeout 600 python -m pytest tests -m gpu -q -x -k "kernel or gradient or relax or clean or smoke" > gpurun_out/pytest_kint.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_kint.log
  timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err
  timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --clock-control none --csv -k regex:k_kint --log-file gpurun_out/launch_kint.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
fi
if [[ $what == mesh ]]; then
  timeout 900 python -m pytest tests/test_mesh_gpu.py -q -x -rf > gpurun_out/pytest_mesh.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mesh.log
  timeout 900 python -m pytest tests/test_refine_gpu.py -q -x -rf > gpurun_out/pytest_refine.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_refine.log
  timeout 600 python scripts/mesh_bench.py 4 5 6 > gpurun_out/mesh_bench.json 2> gpurun_out/mesh_bench.err
  timeout 600 python scripts/mesh_bench.py chain 4 5 6 >> gpurun_out/mesh_bench.json 2>> gpurun_out/mesh_bench.err
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_mesh.csv python scripts/mesh_bench.py 5 > /dev/null 2>&1
fi
if [[ $what == e2e ]]; then
  timeout 900 python -m pytest tests -m gpu -q -x -rf -k "probe or smoke or relax" > gpurun_out/pytest_e2e.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_e2e.log
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err
  python - > gpurun_out/pcie.txt 2>&1 <<'PY'
import torch, time
for mb in (64, 256):
    n = mb << 18
    h = torch.empty(n, dtype=torch.float32).pin_memory(); d = torch.empty(n, device="cuda")
    for direction in ("h2d", "d2h"):
        torch.cuda.synchronize(); t = time.perf_counter()
        for _ in range(5):
            (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
        torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 5
        print(direction, mb, "MB", round(n * 4 / dt / 1e9, 1), "GB/s")
PY
fi
if [[ $what == final ]]; then
  O=gpurun_out/${TAG:-r01h}; mkdir -p $O
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
  timeout 1500 python -m pytest tests -m gpu -q -rf --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
  timeout 900 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
  timeout 900 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
  timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
  B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-kernel-roofline"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $B > $O/ncu_launch.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_sweep' -s 25 -c 1 -o $O/prof_reinit $B > $O/ncu_reinit.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gradient|k_kint|k_probe|k_phi_init|k_count|k_tag|k_nb|k_scatter' -s 7 -c 8 -o $O/prof_other $B > $O/ncu_other.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_sweep|k_gradient|k_kint' -s 26 -c 3 -o $O/prof_c3 python bench.py --config C3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-kernel-roofline > $O/ncu_c3.log 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv python bench.py --config C5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-kernel-roofline > $O/ncu_launch_c5.log 2>&1
fi
if [[ $what == init ]]; then
  timeout 900 python -m pytest tests -m gpu -q -x -rf -k "tables or phi_init or c3 or c5 or smoke or sign or refine or mesh or forced" > gpurun_out/pytest_init.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_init.log
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-kernel-roofline > gpurun_out/bench_init.json 2> /dev/null
  timeout 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline --no-kernel-roofline > gpurun_out/bench_c3_init.json 2> /dev/null
  timeout 300 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-kernel-roofline > gpurun_out/bench_c5_init.json 2> /dev/null
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_init.csv python bench.py --config C3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-kernel-roofline > /dev/null 2>&1
fi
