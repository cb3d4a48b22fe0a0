"""Build variants of libddm.so with compile-time knobs and time the GMRES
solves of scripts/gmres_timing.py (GMRES_CFGS, default "3").

  python scripts/tune_gmres.py base "DDM_AX_UNROLL=8" "DDM_ROW_T=256,DDM_ROW_UPD=16" ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_1812_05087_b200 import build as B
    for v in sys.argv[1:] or ["base"]:
        defs = [] if v == "base" else v.split(",")
        out = f"/tmp/ddm_gvar_{abs(hash(v))}.so"
        B.build(defines=defs, out=out, force=True)
        env = dict(os.environ, DDM_LIB=out, GMRES_CFGS=os.environ.get("GMRES_CFGS", "3"))
        r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "gmres_timing.py"), "3"],
                           env=env, capture_output=True, text=True)
        lines = [ln for ln in r.stdout.splitlines() if "solve" in ln]
        print(f"{v:44s} " + (" | ".join(lines) if lines else "FAILED " + r.stderr[-1500:]),
              flush=True)


if __name__ == "__main__":
    main()
