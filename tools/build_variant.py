"""Build an A/B variant of libfk_b200.so with extra nvcc flags into its own
directory (the product build is paper_2603_09038_b200/build.py):

    python tools/build_variant.py OUTDIR [-DFLAG ...] [--orders 4,6]

Only the listed orders' kernel units get the flags (all by default); load it
with FK_LIB_PATH=OUTDIR/libfk_b200.so."""
import concurrent.futures as cf
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_09038_b200 import build as B  # noqa: E402


def main():
    out = os.path.abspath(sys.argv[1])
    extra = [a for a in sys.argv[2:] if a.startswith("-D")]
    orders = None
    if "--orders" in sys.argv:
        orders = {f"pa_p{o}" for o in sys.argv[sys.argv.index("--orders") + 1].split(",")}
    os.makedirs(out, exist_ok=True)
    units, _ = B.sources()

    def comp(u):
        name, src, ex = u
        o = os.path.join(out, name + ".o")
        fl = extra if (orders is None or name in orders) else []
        cmd = [B.nvcc()] + B.flags() + ex + fl + ["-c", os.path.join(B.CSRC, src), "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(r.stderr)
        return o

    with cf.ThreadPoolExecutor(os.cpu_count()) as ex:
        objs = list(ex.map(comp, units))
    lib = os.path.join(out, "libfk_b200.so")
    subprocess.run([B.nvcc()] + B.ARCH + ["-shared", "-o", lib] + objs + ["-ldl", "-lpthread"], check=True)
    print(lib)


if __name__ == "__main__":
    main()
