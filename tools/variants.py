"""Build and time library variants (compile-time -D knobs) in one GPU call.

    python tools/variants.py build  NAME="-DFOO=1 -DBAR=2" ...   # here
    python tools/variants.py build-rev REV NAME                  # csrc at a git rev
    python tools/variants.py run CONFIG STEPS NAME...             # on the GPU box

Variants go to paper_2403_02997_b200/lib/variants/ (git-ignored); `run`
loads each through TCB_LIBRARY in a fresh process and prints the stage
times of the last step.
"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CSRC = ROOT / "paper_2403_02997_b200" / "csrc"
OUT = ROOT / "paper_2403_02997_b200" / "lib" / "variants"
NVCC = "/usr/local/cuda/bin/nvcc"
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "--extended-lambda", "-Xcompiler", "-fPIC,-fvisibility=hidden,-fopenmp",
         f"-I{ROOT / 'include'}"]


def build(name: str, defs: str, csrc: Path = CSRC):
    obj = ROOT / "paper_2403_02997_b200" / "build" / f"obj_v_{name}"
    obj.mkdir(parents=True, exist_ok=True)
    OUT.mkdir(parents=True, exist_ok=True)
    procs, objs = [], []
    for src in sorted(csrc.glob("*.cu")):
        o = obj / (src.stem + ".o")
        objs.append(str(o))
        procs.append(subprocess.Popen([NVCC, *FLAGS, *defs.split(), "-c", str(src), "-o", str(o)]))
    for p in procs:
        if p.wait() != 0:
            raise SystemExit(f"variant {name}: compile failed")
    lib = OUT / f"libtricount_b200_{name}.so"
    subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart",
                    "static", "-Xcompiler", "-fopenmp", "-o", str(lib), *objs], check=True)
    print("built", lib)


def run(config: str, steps: int, names):
    for name in names:
        lib = OUT / f"libtricount_b200_{name}.so"
        env = dict(os.environ, TCB_LIBRARY=str(lib))
        out = subprocess.run([sys.executable, str(ROOT / "tools" / "profile_step.py"), config,
                              str(steps)], env=env, capture_output=True, text=True)
        lines = [ln for ln in out.stdout.splitlines() if ln.startswith("step")]
        print(f"{name:>12}: {lines[-1] if lines else out.stderr[-400:]}", flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build-rev":
        import tempfile
        tmp = Path(tempfile.mkdtemp())
        subprocess.run(f"git -C {ROOT} archive {sys.argv[2]} paper_2403_02997_b200/csrc include"
                       f" | tar -x -C {tmp}", shell=True, check=True)
        build(sys.argv[3], "", tmp / "paper_2403_02997_b200" / "csrc")
    elif sys.argv[1] == "build":
        for spec in sys.argv[2:]:
            name, _, defs = spec.partition("=")
            build(name, defs.strip('"'))
    else:
        run(sys.argv[2], int(sys.argv[3]), sys.argv[4:])
