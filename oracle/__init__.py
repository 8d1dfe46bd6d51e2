"""CPU oracle for the stage-parallel Radau IIA hot path -- TEST INFRASTRUCTURE ONLY.

Plain numpy/scipy restatement of the reference package (pkg/src/spirk, cited per function) and of
the SPEC/paper pieces the reference has no code for (Q_k elements, the IRK stepper, the stage
transforms, PRESB). Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
it, and only as the checker / the timed CPU baseline -- never as part of the product path.

Pinning: at k = 1 every restated function is checked against golden vectors generated from the
reference itself (tests/golden/make_golden.py -> tests/golden/*.npz). The Q_k generalisation, the
stepper, the transforms and PRESB are pinned by (i) their exact reduction to the reference at k = 1,
(ii) manufactured-solution convergence rates and (iii) the paper's iteration counts (soft).
"""
