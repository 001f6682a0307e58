# 2-pair clusters with A multicast: correctness (kernel + layer tests) then ncu / A/B vs single pairs
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python - <<'PY' > gpurun_out/mc_probe.log 2>&1
import torch
from paper_2601_17111_b200 import llep as L
D, H, E = 512, 512, 4
sizes = [700, 40, 300, 1000]
groups, rb = [], 0
for i, n in enumerate(sizes):
    groups.append((i, rb, n)); rb += (n + 255) // 256 * 256
x = torch.randn(rb, D, device="cuda").to(torch.bfloat16)
w13 = (torch.randn(E, 2 * H, D, device="cuda") / D ** 0.5).to(torch.bfloat16)
act = torch.zeros(rb, H, device="cuda", dtype=torch.bfloat16)
L.grouped_gemm(0, x, w13, groups, H, out=act, pair=True)
torch.cuda.synchronize()
ref = []
for (e, r0, n) in groups:
    gu = x[r0:r0 + n].float() @ w13[e].float().t()
    g, u = gu[:, :H], gu[:, H:]
    ref.append((torch.nn.functional.silu(g) * u, act[r0:r0 + n].float()))
err = max(((a - b).abs().max() / a.abs().max()).item() for a, b in ref)
print("probe max rel err", err)
assert err < 2e-2
PY
echo probe_rc=$?; cat gpurun_out/mc_probe.log | tail -3
if ! grep -q "probe max rel" gpurun_out/mc_probe.log; then echo "probe failed, stopping"; exit 0; fi
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "grouped" > gpurun_out/pytest_mc_kernels.log 2>&1; tail -5 gpurun_out/pytest_mc_kernels.log
timeout 900 python -m pytest tests/test_gpu_layer.py -q -x -k "p1_full or g120_p1_sampled or f3_shapes or multiprocess_p2_p4" > gpurun_out/pytest_mc_layer.log 2>&1; tail -5 gpurun_out/pytest_mc_layer.log
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_bytes.sum,launch__grid_size
for v in 2 1; do LLEP_GEMM_MC=$v timeout 300 ncu --metrics $M --clock-control none -k regex:grouped_gemm -c 2 --csv python tools/gemm_bench.py --layout hot --variants cta2 --iters 1 > gpurun_out/mc_hot_$v.csv 2>&1; done
for v in 1 2; do LLEP_GEMM_MC=$v timeout 300 ncu --metrics $M --clock-control none -k regex:grouped_gemm_2cta -s 12 -c 2 --csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-distinct --no-backward --no-emulation > gpurun_out/mc_g120_$v.csv 2>&1; done
timeout 300 python tools/fwd_ab.py LLEP_GEMM_MC 1 2 --config g120 --hot 95 --secs 4 > gpurun_out/ab_mc.jsonl 2>&1
timeout 300 python tools/fwd_ab.py LLEP_GEMM_MC 1 2 --config q3 --hot 95 --secs 3 >> gpurun_out/ab_mc.jsonl 2>&1
cat gpurun_out/ab_mc.jsonl | cut -c1-400
