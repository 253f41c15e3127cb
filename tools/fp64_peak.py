"""cuBLAS DGEMM peak on the box (FP64 roofline denominator; MEASURED_PEAKS.json has no FP64 entry)."""
import json, torch
def main():
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); a @ b; e.record(); e.synchronize(); best = min(best, s.elapsed_time(e))
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20): a @ b
    e.record(); e.synchronize(); sus = s.elapsed_time(e) / 20
    print(json.dumps({"dgemm_n": n, "burst_tflops": 2 * n**3 / best / 1e9, "sustained_tflops": 2 * n**3 / sus / 1e9}))
if __name__ == "__main__":
    main()
