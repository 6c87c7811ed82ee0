"""Developer tool: build a variant of the library with extra -D flags on hs_solve.cu (tuning
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
    obj = os.path.join(out_dir, f"hs_solve_{name}.o")
    src = os.path.join(B.CSRC, "hs_solve.cu")
    subprocess.run([B._nvcc()] + B._flags() + defs + ["-x", "cu", "-c", src, "-o", obj], check=True)
    objs = [os.path.join(B.BUILD, os.path.basename(s) + ".o") for s in B.sources() if not s.endswith("hs_solve.cu")]
    out = os.path.join(out_dir, f"{name}.so")
    subprocess.run([B._nvcc()] + B.ARCH + ["-ccbin", B.HOST_CXX, "-shared", "-o", out] + objs + [obj, "-lcudart_static", "-ldl"], check=True)
    print(out)

if __name__ == "__main__":
    main()
