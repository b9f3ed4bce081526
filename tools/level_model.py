"""Developer tool: predict a query's device time from its compiled level schedule (CPU only, no GPU).

    python tools/level_model.py [config ...] [--flags-extra N]

Level time model (measured per-width level times on one B200 with tools/level_curve.py):
whole waves of 5 x 148 bootstraps at 12.7 ms, plus one tail wave whose kernel depends on its width --
6-CTA clusters (<= 24) 2.7 ms, 2-CTA clusters (<= 74) 2.9 ms, 6 warp groups per bootstrap (<= 148) 3.5 ms,
else ceil(tail / 148) bootstraps per SM at 4.8 / 6.1 / 8.0 / 10.3 / 12.7 ms.  The key switch (< 1 %) is ignored.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12761_b200 import _lib as L  # noqa: E402
from paper_2506_12761_b200 import api as A  # noqa: E402
from synth import make_workload  # noqa: E402

WAVE, T_WAVE = 740, 12.7
T_B = {1: 4.8, 2: 6.1, 3: 8.0, 4: 10.3, 5: 12.7}


def level_ms(width: int) -> float:
    if width == 0:
        return 0.0
    full, tail = divmod(width, WAVE)
    t = full * T_WAVE
    if tail:
        t += 2.7 if tail <= 24 else 2.9 if tail <= 74 else 3.5 if tail <= 148 else T_B[-(-tail // 148)]
    return t


def level_widths(m) -> list:
    h = ctypes.c_void_p()
    L.check(L.lib().vlp_program_create(None, ctypes.byref(m), 0, m.M, ctypes.byref(h)))
    info = L.VlpProgramInfo()
    L.check(L.lib().vlp_program_get_info(h, ctypes.byref(info)))
    ws = []
    for lv in range(info.levels):
        nb, nk = ctypes.c_uint64(), ctypes.c_uint64()
        L.check(L.lib().vlp_program_level_jobs(h, lv, None, ctypes.byref(nb), None, ctypes.byref(nk)))
        ws.append(nb.value)
    L.lib().vlp_free_program(h)
    return ws


def main():
    args = sys.argv[1:]
    extra = 0
    if "--flags-extra" in args:
        i = args.index("--flags-extra")
        extra = int(args[i + 1])
        del args[i:i + 2]
    for cfg in [int(a) for a in args] or [1, 2, 6, 7, 8, 9]:
        wl = make_workload(cfg)
        m = A.meta(wl.mode, wl.M, wl.l_I, wl.l_S, wl.d, wl.flags | extra)
        ws = level_widths(m)
        print(f"config {cfg} ({wl.name}): {len(ws)} levels, {sum(ws)} BR, predicted {sum(map(level_ms, ws)):.0f} ms")


if __name__ == "__main__":
    main()
