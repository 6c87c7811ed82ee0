"""Developer tool: build a variant of the library with extra -D flags on hs_solve.cu / hs_ddm.cu / hs_kernels.cu (tuning
experiments). Usage: python tools/build_variant.py NAME -DHS_NS_FWD=2 ...  ->  _variants/NAME.so,
selected at run time with HS_LIB_PATH."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2003_02585_b200 import build as B

def main():
    name, defs = sys.argv[1], sys.argv[2:]
    B.build()
    out_dir = os.path.join(ROOT, "paper_2003_02585_b200", "_variants")
    os.makedirs(out_dir, exist_ok=True)
    # the -D flags apply to the solve kernels and to the host item builder
    var = ["hs_solve.cu", "hs_ddm.cu", "hs_kernels.cu"]
    vobjs = []
    for f in var:
        obj = os.path.join(out_dir, f"{f}_{name}.o")
        subprocess.run([B._nvcc()] + B._flags() + defs + ["-x", "cu", "-c", os.path.join(B.CSRC, f), "-o", obj], check=True)
        vobjs.append(obj)
    objs = [os.path.join(B.BUILD, os.path.basename(s) + ".o") for s in B.sources() if os.path.basename(s) not in var]
    out = os.path.join(out_dir, f"{name}.so")
    subprocess.run([B._nvcc()] + B.ARCH + ["-ccbin", B.HOST_CXX, "-shared", "-o", out] + objs + vobjs + ["-lcudart_static", "-ldl"], check=True)
    print(out)

if __name__ == "__main__":
    main()
