"""Read the raw page of an ncu capture: a .ncu-rep (via `ncu -i`) or the CSV the GPU box
exported from it (`ncu -i REP --page raw --csv`, optionally gzipped) when the report itself
is too large to bring back."""
import csv
import gzip
import subprocess


def raw_rows(path):
    if path.endswith(".csv.gz"):
        with gzip.open(path, "rt") as f:
            text = f.read()
    elif path.endswith(".csv"):
        with open(path) as f:
            text = f.read()
    else:
        text = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(text.splitlines()))
