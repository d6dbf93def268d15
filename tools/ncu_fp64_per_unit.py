"""FP64 thread-instructions per unit of work from an ncu --set full capture:
(dadd + dmul + dfma per elapsed cycle, summed over SMSPs) x elapsed cycles
/ units.  Verifies the per-unit work W a roofline is quoted with.

    python tools/ncu_fp64_per_unit.py <rep> <units>
"""
import csv
import io
import subprocess
import sys


def main(path, units):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, val = rows[0], rows[2]
    get = {h: v for h, v in zip(hdr, val)}
    per_cycle = sum(float(get[f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed"])
                    for op in ("dadd", "dmul", "dfma"))
    cycles = float(get["smsp__cycles_elapsed.avg"]) if "smsp__cycles_elapsed.avg" in get else \
        float(get["gpu__time_duration.sum"]) * 1e-9 * float(get["sm__cycles_elapsed.avg.per_second"])
    total = per_cycle * cycles
    print(f"{path}: {total:.4g} FP64 thread-instructions, {total / units:.2f} per unit "
          f"({units:g} units)")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]))
