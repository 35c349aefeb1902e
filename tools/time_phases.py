"""Per-kernel device times of one R(u) at config 2 via ncu-free event pairs:
times R, then R with the phase kernels launched individually through the
library is not possible from Python, so this reports the whole-R time and
the ncu launch list is used for shares."""
