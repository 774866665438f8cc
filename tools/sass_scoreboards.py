"""Decode the scoreboard fields of a kernel's SASS control words (run here, no GPU).

    python tools/sass_scoreboards.py build/obj/spmv_f64.cu.o '<mangled kernel name>' [--all]

sm_100a instructions are 128 bits; bits 105..125 of each hold the scheduling
control: stall count (4 bits), yield, the write barrier an instruction sets
(3 bits, 7 = none), the read barrier (3 bits) and the 6-bit mask of barriers
it waits for.  ptxas has six barriers ("scoreboards") per warp, and a wait
drains *everything* outstanding on a barrier — so which loads share one
decides what a use really waits for (the sliced kernels'
metadata loads and the tiled kernel's two register batches).  Prints
index, address, instruction, `W<n>` (sets write barrier n), `R<n>`, and
`wait=<barriers>`; by default only memory instructions, waits and branches.
"""
import re
import subprocess
import sys


def decode(obj, fun):
    out = subprocess.run(["cuobjdump", "-sass", "-fun", fun, obj], capture_output=True,
                         text=True).stdout.split("\n")
    first = re.compile(r"^\s+/\*([0-9a-f]{4,5})\*/\s+(.*?);\s+/\* 0x([0-9a-f]{16}) \*/")
    second = re.compile(r"^\s+/\* 0x([0-9a-f]{16}) \*/")
    ins, i = [], 0
    while i < len(out):
        m = first.match(out[i])
        m2 = second.match(out[i + 1]) if m and i + 1 < len(out) else None
        if m2:
            hi = int(m2.group(1), 16)
            ins.append((m.group(1), m.group(2), (hi >> 41) & 0xf, (hi >> 46) & 7, (hi >> 49) & 7,
                        (hi >> 52) & 0x3f))
            i += 2
        else:
            i += 1
    return ins


if __name__ == "__main__":
    everything = "--all" in sys.argv
    for k, (addr, text, stall, wb, rb, wm) in enumerate(decode(sys.argv[1], sys.argv[2])):
        keep = everything or wm or any(t in text for t in ("LDG", "STG", "LDS", "STS", "BLKPF",
                                                            "BLKCP", "BRA", "SYNCS"))
        if keep:
            flags = (f"W{wb}" if wb != 7 else "  ") + (f" R{rb}" if rb != 7 else "   ")
            if wm:
                flags += " wait=" + "".join(str(b) for b in range(6) if wm >> b & 1)
            print(k, addr, text[:78], flags)
