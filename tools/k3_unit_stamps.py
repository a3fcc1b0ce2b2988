"""Where does the single-expert unit kernel spend its time?  Builds a
diagnostic libspmoe variant with -DSPMOE_UNIT_STAMPS (per-CTA globaltimer
stamps at the kernel's phase boundaries; the product build has none), runs
one Mixtral expert (T tokens) on cold slots and prints the median over CTAs
and calls of each phase, in microseconds from the earliest CTA entry:

  0 entry  1 setup done (barriers, TMEM)  2 first up stage landed (MMA)
  3 last up MMA issued  4 h written (epilogue)  5 first down MMA may issue
  6 last W2 load issued (producer)  7 last y tile stored (epilogue)

Usage: python tools/k3_unit_stamps.py [T] [iters] [NY (down-phase y accumulators)]
(the stream without math for comparison: tools/probes/tma_stream.cu unit)."""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch


def build_variant(out: Path, ny: int = 2) -> Path:
    from paper_2510_10302_b200 import build as B

    srcs = [str(s) for s in B.SOURCES if s.exists()]
    cmd = [B.nvcc_path(), *B.ARCH_FLAGS, "-O3", "-lineinfo", "-std=c++17", "-DSPMOE_UNIT_STAMPS", f"-DSPMOE_UNIT_NY={ny}", "-Xcompiler",
           "-fPIC,-O3", "-shared", "-o", str(out), *srcs, "-lpthread"]
    out.parent.mkdir(exist_ok=True)
    subprocess.run(cmd, check=True)
    return out


def main(T=1, iters=12, ny=2):
    from paper_2510_10302_b200 import _native

    lib_path = build_variant(ROOT / "_variants" / f"unit_stamps_ny{ny}.so", ny)
    _native.LIB_PATH = lib_path
    from paper_2510_10302_b200 import kernels as K

    lib = _native.load()
    H, F, S = 4096, 14336, 8
    dev = "cuda"
    pool = torch.empty((S, 3 * F * H), dtype=torch.bfloat16, device=dev)
    K.fill_normal_(pool, 7, 0, 0.02)
    g = torch.Generator().manual_seed(T)
    x = torch.randn((T, H), generator=g).to(torch.bfloat16).to(dev)
    idx = torch.zeros((T, 1), dtype=torch.int32, device=dev)
    off, perm, inv = K.moe_permute(idx, 1)
    y = torch.empty((T, H), dtype=torch.float32, device=dev)
    xp = torch.empty((T, H), dtype=torch.bfloat16, device=dev)
    wsu = torch.zeros((K.tc_units_workspace_floats(T, H, F),), dtype=torch.float32, device=dev)
    st = torch.zeros((148, 8), dtype=torch.int64, device=dev)
    import ctypes

    assert lib.spmoe_debug_unit_stamps(ctypes.c_void_p(st.data_ptr())) == 0
    rows = []
    for i in range(iters + 2):
        st.zero_()
        torch.cuda.synchronize()
        K.expert_ffn_tc_units(pool, [i % S], 1, x, F, 1, off, perm, T, xp, None, y, wsu)
        torch.cuda.synchronize()
        if i < 2:
            continue
        a = st[:112].cpu().numpy().astype(np.float64)
        t0 = a[:, 0].min()
        rows.append((a - t0) / 1e3)
    r = np.stack(rows)  # [calls, cta, 8] us
    names = ["entry", "setup", "up1st", "upMMAend", "h_ready", "dn1st", "ldLast", "yEnd"]
    med = np.median(r, axis=(0, 1))
    mx = np.median(r.max(axis=1), axis=0)
    print(f"T={T} NY={ny}: median over CTAs (max over CTAs) us from first entry")
    for n, m, x_ in zip(names, med, mx):
        print(f"  {n:9s} {m:7.2f} ({x_:7.2f})")
    d = r[..., 5] - r[..., 3]
    print(f"  up->down transition (MMA idle): median {np.median(d):.2f} us; kernel span {np.median(r[..., 7].max(axis=1)):.2f} us")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(int(a[0]) if a else 1, int(a[1]) if len(a) > 1 else 12, int(a[2]) if len(a) > 2 else 2)
