"""Write profiles/traffic.json entries (DRAM bytes per launch of the dominant kernel)
from ncu --set full captures.  Usage:
    python scripts/traffic_json.py KEY REPORT.ncu-rep KERNEL_REGEX [KEY REPORT REGEX ...]
KEY = "<config>/<rows per GPU>/<algo>" as bench.py looks it up."""
import csv
import io
import json
import os
import re
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def dram_bytes(report, kernel_regex):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    ki = h.index("Kernel Name")
    for r in rows[2:]:
        if re.search(kernel_regex, r[ki]):
            get = lambda m: float(r[h.index(m)].replace(",", "")) * SCALE[u[h.index(m)]]  # noqa: E731
            return {"dram_bytes_read": get("dram__bytes_read.sum"), "dram_bytes_write": get("dram__bytes_write.sum"),
                    "kernel": r[ki][:80], "source": os.path.basename(report) + " (ncu --set full, one launch)"}
    raise SystemExit(f"no kernel matching {kernel_regex} in {report}")


def main(args):
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    for key, rep, rx in zip(args[0::3], args[1::3], args[2::3]):
        data[key] = dram_bytes(rep, rx)
        print(key, data[key])
    json.dump(data, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:])
