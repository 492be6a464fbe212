"""Per-CUDA-source-line warp-stall samples and executed instructions of one
kernel in an ncu report (profiling helper):
    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [N]"""
import csv, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kern}", "--launch-count", "1"], capture_output=True, text=True).stdout
fname, data = None, []
for r in csv.reader(out.splitlines()):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif len(r) > 8 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            data.append((float(r[4]), float(r[7]), f"{fname}:{r[0]}", r[1][:100]))
        except ValueError:
            pass
ts, ti = sum(d[0] for d in data) or 1, sum(d[1] for d in data) or 1
print(f"samples {ts:.0f}  instructions {ti:.0f}")
for d in sorted(data, reverse=True)[:top]:
    print(f"{100 * d[0] / ts:5.1f}% stall {100 * d[1] / ti:5.1f}% inst  {d[2]:>18}  {d[3]}")
