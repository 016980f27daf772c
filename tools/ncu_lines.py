"""Per-CUDA-source-line hot spots of an ncu report (needs -lineinfo and --import-source):
warp-stall samples and executed warp instructions, top N lines."""
import csv, io, subprocess, sys


def main(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows, fname, hdr = [], None, None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "" or r[0] == "Function Name":
            continue
        d = dict(zip(hdr, r))
        try:
            samp = int(d["Warp Stall Sampling (All Samples)"])
            inst = int(d["Instructions Executed"])
        except (ValueError, KeyError):
            continue
        rows.append((samp, inst, f"{fname}:{r[0]}", r[1].strip()[:90]))
    ts = sum(x[0] for x in rows) or 1
    ti = sum(x[1] for x in rows) or 1
    print(f"total samples {ts}, warp instructions {ti}")
    for samp, inst, loc, src in sorted(rows, reverse=True)[:top]:
        print(f"{samp / ts:6.1%} stall  {inst / ti:6.1%} inst  {loc:22s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
