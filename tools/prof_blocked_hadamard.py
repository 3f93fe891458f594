"""Tensor-core check for the blocked-Hadamard formulation of the k = 14 FWHT (tools only).
H_16384 = H_128 (x) H_128, so one basis-row's transform is two 128x128x128 GEMMs (X -> H X H).
Times the cuBLAS GEMMs that formulation needs, (rows*128 x 128) @ (128 x 128), in bf16 and TF32,
and prints the implied time per basis-row against the CUDA-core butterfly cost
(229,376 adds at the measured 36.7 Tadd/s) and the current kernel (~123 ms per 1024 rows x 8192 bases)."""
import torch

torch.backends.cuda.matmul.allow_tf32 = True
H = torch.ones(1, 1, device="cuda")
for _ in range(7):
    H = torch.cat([torch.cat([H, H], 1), torch.cat([H, -H], 1)], 0)  # Sylvester H_128
rows = 8192                                      # basis-rows per GEMM batch
for dt, name in ((torch.bfloat16, "bf16"), (torch.float32, "tf32")):
    X = torch.randn(rows * 128, 128, device="cuda").to(dt)
    Hd = H.to(dt)
    for _ in range(3):
        Y = X @ Hd
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        Y = X @ Hd
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    flops = 2.0 * rows * 128 * 128 * 128
    per_row_ns = 2 * ms * 1e6 / rows             # two GEMMs per basis-row (H X and X H)
    print(f"{name}: {flops / ms / 1e9:.0f} TFLOP/s on K = N = 128; {per_row_ns:.1f} ns per basis-row "
          f"({3 * per_row_ns:.1f} ns with the 3-term split fp32 accuracy needs); "
          f"CUDA-core butterflies at the measured add peak: {229376 / 36.7e12 * 1e9:.1f} ns; "
          f"current kernel: {123e-3 / (1024 * 8192) * 1e9:.1f} ns per basis-row (chip-wide)")
