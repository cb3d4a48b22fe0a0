"""ORACLE — test infrastructure only.

A plain, slow, obviously correct CPU implementation (numpy, fp64) of what the
FMM-DDM hot path computes, written from the paper (Rezaei et al., arXiv
1812.05087, /root/reference/PAPER.md, cited as P:line) and the readings in
DESIGN.md §2.  It shares no code with the CUDA path
(`paper_1812_05087_b200/`) and neither imports the other; only the seeded
input generators in `synth/` serve both.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import or execute anything in this package.  The
product path must never route through it.

Modules
-------
elastic  dense Crouch–Starfield influence matrix (Eq.(final_sigs)),
         direct matvec, far-field loads
tree     Morton keys by bit loop, pointer quad-tree, brute-force U/V lists
         
gmres    dense restarted GMRES with CGS2
sif      Olson's SIF formula, Eq.(SIF)
history  direct history double sum of Eq.(final_sigs)-(final_pp)
poro     poroelastic continuous-source kernel — see its header
         for the pin status.
"""
