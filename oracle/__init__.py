"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference's CDP training-step numerics, used as the
parity checker for the sm_100a path and as the CPU baseline in bench.py.
Only `tests/`, `__graft_entry__.smoke()` and `bench.py` (cpu_baseline leg and
`--impl reference`) may import this package; the product
(`paper_2403_08837_b200`) never does and fails loudly without its CUDA
library instead of falling back here.

* `oracle/cdp_oracle.c`   value+grad kernels, bit-identical to the
                          reference's `_kernels.pyx` (pinned by
                          tests/golden/ vectors made from the reference);
* `oracle/engine.py`      `_advance` / `run_experiment` restatement
                          (ref `training/engine.py:66-215`) and the task
                          generators (ref `training/models.py:173-225`);
* `oracle/_ref/`          the reference's own Cython kernel compiled from
                          /root/reference by `oracle/build.py`.
"""
