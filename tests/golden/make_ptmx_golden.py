"""Writes tests/golden/ptmx_v1_3x2.ptmx byte by byte from the PTMX v1 layout
in the reference's io.hpp:23-51 (magic "PTMX", u32 version 1, u64 rows,
u64 cols, f64 dt, f64 t0, column-major f64 payload), independently of
paper_2103_01983_b200.bundle. Run once; the output is committed."""
import os
import struct

HERE = os.path.dirname(os.path.abspath(__file__))
rows, cols = 3, 2
# matrix [[1, 4], [2, 5], [3, 6]] * 0.5 ; column-major payload 0.5, 1, 1.5, 2, 2.5, 3
payload = [0.5 * (k + 1) for k in range(rows * cols)]
with open(os.path.join(HERE, "ptmx_v1_3x2.ptmx"), "wb") as f:
    f.write(b"PTMX")
    f.write(struct.pack("<I", 1))
    f.write(struct.pack("<Q", rows))
    f.write(struct.pack("<Q", cols))
    f.write(struct.pack("<d", 1e-3))
    f.write(struct.pack("<d", 0.25))
    for v in payload:
        f.write(struct.pack("<d", v))
