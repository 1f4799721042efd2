"""Decode the scheduling control bits (stall, yield, barriers) of cuobjdump -sass output.
usage: cuobjdump -sass -fun NAME lib.so | python tools/sass_ctrl.py [start_addr end_addr]"""
import re
import sys

lines = sys.stdin.read().splitlines()
lo = int(sys.argv[1], 16) if len(sys.argv) > 2 else 0
hi = int(sys.argv[2], 16) if len(sys.argv) > 2 else 1 << 62
i = 0
while i < len(lines):
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);\s*/\* (0x[0-9a-f]+) \*/", lines[i])
    if m and i + 1 < len(lines):
        m2 = re.match(r"\s*/\* (0x[0-9a-f]+) \*/", lines[i + 1])
        addr = int(m.group(1), 16)
        if m2 and lo <= addr <= hi:
            hiw = int(m2.group(1), 16)
            ctrl = hiw >> 41
            stall = ctrl & 0xF
            yld = (ctrl >> 4) & 1
            wbar = (ctrl >> 5) & 7
            rbar = (ctrl >> 8) & 7
            wmask = (ctrl >> 11) & 0x3F
            reuse = (ctrl >> 17) & 0xF
            print(f"{addr:05x} S{stall:2d} Y{yld} W{wbar if wbar != 7 else '-'} R{rbar if rbar != 7 else '-'} "
                  f"M{wmask:02x}  {m.group(2).strip()}")
        i += 2
    else:
        i += 1
