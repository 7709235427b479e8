"""Write profiles/ncu_k3_<config>.json from an ncu --set full capture of one
tensor-core K3 launch: DRAM bytes (read + write) of that launch, which
bench.py reports as roofline.traffic next to the algorithmic bytes.

usage: python profiles/ncu_k3_traffic.py <report.ncu-rep> <config>
"""
import csv
import io
import json
import os
import subprocess
import sys


def main():
    rep, name = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]

    def val(r, key):
        v = float(r[hdr.index(key)].replace(",", ""))
        u = units[hdr.index(key)]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(u, 1)
        return v * scale

    r = [x for x in rows[2:] if "expert_ffn_t" in x[hdr.index("Kernel Name")]][0]
    kname = r[hdr.index("Kernel Name")]
    rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
    t = val(r, "gpu__time_duration.sum")
    out = {"config": name, "kernel": kname, "report": os.path.basename(rep),
           "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
           "duration_s_under_ncu": t, "dram_GBps_under_ncu": (rd + wr) / t / 1e9,
           "note": "one launch, ncu --set full --clock-control none (serialised, cache-control all): "
                   "its time is not a bench number; traffic is compared with the launch's algorithmic bytes"}
    # algorithmic bytes of that launch: the number of expert images it streamed
    # is the nearest integer to DRAM reads / image bytes (activations and
    # partials are < 2% of an image at these shapes)
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2603_09983_b200.configs import CONFIGS
    w = CONFIGS[name]
    img = 3 * w.d_model * w.d_ffn * 2
    n_img = max(1, round(rd / img))
    out.update({"expert_image_bytes": img, "images_streamed_in_launch (inferred)": n_img,
                "algorithmic_bytes_of_launch": n_img * img, "traffic_over_algorithmic": round((rd + wr) / (n_img * img), 4)})
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"ncu_k3_{name}.json")
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
