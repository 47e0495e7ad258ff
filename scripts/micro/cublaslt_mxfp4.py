"""Probe: the library's block-scaled FP4 GEMM on this B200 next to k_gemm_mxf4_2sm. torch 2.11 exposes
no MXFP4 (E2M1 + UE8M0 per 32) scaled_mm, so the reference is cuBLASLt NVFP4 (E2M1 x E2M1 with E4M3
scales per 16 along K — the same FP4 tensor-core rate, twice the scale factors) through
F.scaled_mm, plus MXFP8 (1x32) for context. Device times from torch.profiler (L2 flushed before
each rep). Random codes / scales: the timing does not depend on the values.
Usage: python scripts/micro/cublaslt_mxfp4.py"""
import sys

import torch

sys.path.insert(0, ".")
try:
    import paper_2604_02525_b200 as ah
except Exception:  # noqa: BLE001
    ah = None

SHAPES = [(8192, 8192, 8192), (16384, 2048, 2048), (16384, 8192, 2048), (16384, 2048, 8192),
          (2048, 8192, 16384), (16384, 512, 2048), (16384, 4096, 4096), (16384, 14336, 4096),
          (16384, 4096, 14336)]


def blocked_scales(rows, k, dev):
    # (rows, k/32) e8m0 scales in the 128x4 swizzled tile layout cuBLASLt expects, flattened
    r = (rows + 127) // 128 * 128
    c = (k // 32 + 3) // 4 * 4
    s = torch.randint(120, 124, (r, c), dtype=torch.uint8, device=dev)
    return s.view(torch.float8_e8m0fnu).reshape(-1)


def main():
    dev = torch.device("cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    print(torch.__version__, torch.cuda.get_device_name())
    for (M, N, K) in SHAPES:
        F = torch.nn.functional
        a = torch.randint(0, 256, (M, K // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
        b = torch.randint(0, 256, (N, K // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
        sa = torch.full((M, K // 16), 1.0, device=dev).to(torch.float8_e4m3fn)
        sb = torch.full((K // 16, N), 1.0, device=dev).to(torch.float8_e4m3fn)
        try:
            f = lambda: F.scaled_mm(a, b.t(), [sa], [F.ScalingType.BlockWise1x16], [sb],  # noqa: E731
                                    [F.ScalingType.BlockWise1x16], [F.SwizzleType.SWIZZLE_32_4_4],
                                    [F.SwizzleType.SWIZZLE_32_4_4], None, torch.bfloat16)
            f()
        except Exception as e:  # noqa: BLE001
            print(f"{M}x{N}x{K}: NVFP4 scaled_mm failed: {type(e).__name__}: {str(e)[:600]}")
            continue
        a8 = torch.randn(M, K, device=dev).to(torch.float8_e4m3fn)
        b8 = torch.randn(N, K, device=dev).to(torch.float8_e4m3fn)
        s8a = torch.full((M, K // 32), 1.0, device=dev).to(torch.float8_e8m0fnu)
        s8b = torch.full((K // 32, N), 1.0, device=dev).to(torch.float8_e8m0fnu)
        f8 = lambda: F.scaled_mm(a8, b8.t(), [s8a], [F.ScalingType.BlockWise1x32], [s8b],  # noqa: E731
                                 [F.ScalingType.BlockWise1x32], [F.SwizzleType.SWIZZLE_32_4_4],
                                 [F.SwizzleType.SWIZZLE_32_4_4], None, torch.bfloat16)
        try:
            _, t8 = prof_time(f8, flush)
            fp8 = f" | MXFP8 {2 * M * N * K / t8 / 1e6:6.0f}"
        except Exception as e:  # noqa: BLE001
            fp8 = f" | MXFP8 failed {str(e)[:100]}"
        names, t = prof_time(f, flush)
        ours = ""
        if ah is not None:
            ca = torch.randint(0, 256, (M, K // 2), dtype=torch.uint8, device=dev)
            cb = torch.randint(0, 256, (N, K // 2), dtype=torch.uint8, device=dev)
            ea = torch.randint(118, 122, (M, K // 32), dtype=torch.uint8, device=dev)
            eb = torch.randint(118, 122, (N, K // 32), dtype=torch.uint8, device=dev)
            _, t2 = prof_time(lambda: ah.debug_gemm_mxf4(ca, ea, cb, eb, out_dtype=torch.bfloat16), flush,
                              only="k_gemm_mxf4")
            ours = f" | ours {t2:8.1f} us {2 * M * N * K / t2 / 1e6:6.0f} TFLOP/s"
        print(f"M={M:6d} N={N:6d} K={K:6d}  NVFP4 {t:8.1f} us {2 * M * N * K / t / 1e6:6.0f} TFLOP/s{ours}{fp8}  [{names}]")


def prof_time(f, flush, only=None):
    """Median device time (us) of the kernels f launches (torch.profiler), L2 flushed before each."""
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(10):
            flush.zero_()
            torch.cuda._sleep(1000)
            f()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
          and "elementwise" not in e.name and "sleep" not in e.name.lower() and "fill" not in e.name.lower()
          and (only is None or only in e.name)]
    names = sorted({e.name[:60] for e in ev})
    per = sorted(e.device_time for e in ev)
    return ",".join(names), per[len(per) // 2] if per else float("nan")

if __name__ == "__main__":
    main()
