"""Writes the Philox words of tests/golden/epoch_perm_example.txt.  Calls only oracle/ (the
Philox4x32-10 primitive, itself pinned by the Random123 KAT vectors); the key assembly and the
resulting orders in that file are derived by hand from these words (see its header)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import sampling as OS  # noqa: E402

for epoch in (0, 3):
    for v in range(6):
        w = OS.philox4x32([v, 0, (1 << 28) | ((epoch & 0xFFFFF) << 8), 0], [1, 0])
        print(f"words 1 {epoch} {v} {w[0]:08x} {w[1]:08x}")
