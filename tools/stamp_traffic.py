"""Stamp profiles/attn_traffic.json from an ncu --set full capture of k_attn at cfg3:
the DRAM bytes of the launch and the kernel-source hash of the build it measured
(bench.py uses it only while the sources are unchanged). Tooling, not product.
usage: python tools/stamp_traffic.py <report.ncu-rep> <capture description> [sha]"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import source_sha  # noqa: E402

rep, desc = sys.argv[1], sys.argv[2]
sha = sys.argv[3] if len(sys.argv) > 3 else source_sha()
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units, v = rows[0], rows[1], rows[2]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def get(name):
    i = h.index(name)
    return int(round(float(v[i]) * scale[units[i]]))


rec = [{"workload": "cfg3", "shard_of": 1, "kernel": "k_attn",
        "dram_bytes_read": get("dram__bytes_read.sum"), "dram_bytes_write": get("dram__bytes_write.sum"),
        "source_sha": sha, "capture": desc}]
(ROOT / "profiles" / "attn_traffic.json").write_text(json.dumps(rec, indent=1) + "\n")
print(json.dumps(rec, indent=1))
