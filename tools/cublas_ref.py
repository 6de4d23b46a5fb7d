"""Reference point only (not on any product path): cuBLASLt int8 GEMM
(torch._int_mm) and cuBLAS bf16 at 8192^3 on this box."""
import torch

n = 8192
a = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda")
b = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()


def bench(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


try:
    ms = bench(lambda: torch._int_mm(a, b))
    print(f"cuBLASLt int8 (_int_mm) {n}^3: {ms:.3f} ms = {2 * n ** 3 / ms / 1e9:.0f} TOPS")
except Exception as e:  # noqa: BLE001
    print("int_mm failed", e)
x = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
y = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
ms = bench(lambda: x @ y)
print(f"cuBLAS bf16 {n}^3: {ms:.3f} ms = {2 * n ** 3 / ms / 1e9:.0f} TFLOPS")
