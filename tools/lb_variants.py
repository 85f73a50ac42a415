"""Build variants of libwpb200.so that differ only in chain_lb build-time switches
(wp_lb.cuh LB_* macros), for A/B timing on the GPU box:

    python tools/lb_variants.py build NAME=-DLB_EG=2,-DLB_FFMA2=0 ...
    python tools/lb_variants.py build NAME@REV=...    # wp_lb.cu/.cuh (and wp_internal.h) as of git REV
    python tools/lb_variants.py build NAME%wp_fir_tc.cu=-DX   # a variant of another translation unit
    python tools/lb_variants.py run cfg3          # on the GPU: every built variant, tools/trace_lb.py timing

Variants land in tools/variants/<NAME>/libwpb200.so (git-ignored, travels with gpurun)."""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "tools", "variants")


def build(specs):
    from paper_2504_08624_b200 import _build as b

    b.build_native()
    objs = sorted(glob.glob(os.path.join(b.OBJ_DIR, "*.o")))
    for spec in specs:
        name, _, flags = spec.partition("=")
        name, _, srcfile = name.partition("%")  # NAME%wp_fir_tc.cu=...: a variant of another source file
        srcfile = srcfile or "wp_lb.cu"
        name, _, rev = name.partition("@")
        flags = [f for f in flags.split(",") if f]
        out = os.path.join(VDIR, name)
        os.makedirs(out, exist_ok=True)
        obj = os.path.join(out, srcfile[:-3] + ".o")
        src = os.path.join(b.CSRC, srcfile)
        if rev:
            # the chain kernel sources of an older revision, next to the current other headers
            sdir = os.path.join(out, "csrc")
            subprocess.run(["cp", "-r", b.CSRC, sdir + "_tmp"], check=True)
            subprocess.run(["rm", "-rf", sdir], check=True)
            os.rename(sdir + "_tmp", sdir)
            for f in ("wp_lb.cu", "wp_lb.cuh", "wp_internal.h", "wp_tc.cuh"):
                txt = subprocess.run(["git", "show", f"{rev}:paper_2504_08624_b200/csrc/{f}"], cwd=ROOT,
                                     capture_output=True, text=True, check=True).stdout
                open(os.path.join(sdir, f), "w").write(txt)
            src = os.path.join(sdir, "wp_lb.cu")
        cmd = [b.NVCC, *b.ARCH, *b.FLAGS, *flags, "-I", b.CSRC, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise SystemExit(r.stderr)
        link = [o for o in objs if not o.endswith(os.path.basename(obj))] + [obj]
        r = subprocess.run([b.NVCC, *b.ARCH, "-shared", "-o", os.path.join(out, "libwpb200.so"), *link, "-lpthread"],
                           capture_output=True, text=True)
        if r.returncode:
            raise SystemExit(r.stderr)
        with open(os.path.join(out, "flags.txt"), "w") as fh:
            fh.write(" ".join(flags) + "\n")
        print("built", name, flags)


def run(cfg):
    names = sorted(os.listdir(VDIR)) if os.path.isdir(VDIR) else []
    for name in ["default"] + names:
        env = dict(os.environ)
        if name != "default":
            env["WP_LIB"] = os.path.join(VDIR, name, "libwpb200.so")
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "trace_lb.py"), cfg], capture_output=True,
                           text=True, env=env, timeout=300)
        lines = [l for l in r.stdout.splitlines() if "ms per pass" in l or "->" in l]
        print(f"== {name}: " + (open(os.path.join(VDIR, name, "flags.txt")).read().strip() if name != "default" else ""))
        print("\n".join(lines) if lines else r.stderr[-2000:])


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    else:
        run(sys.argv[2] if len(sys.argv) > 2 else "cfg3")
