"""profiles/traffic.json from the ncu --set full summaries of one sort per
config (profiles/capture_cfgs.sh -> <tag>_ncu_cfgC.json): per bench kernel
name, dram__bytes_read.sum + dram__bytes_write.sum of its longest launch;
k_wide_scatter = the mean of its two longest launches (the root's bulk-copy
variant and level 1's register-staged one), matching bench.py's per-launch
average.

    python profiles/make_traffic.py r02 > profiles/traffic.json
"""
import json
import re
import sys

NAMES = [(r"k_wide_scatter", "k_wide_scatter"), (r"k_wide_count", "k_wide_count"),
         (r"k_local_w", "k_local_w"), (r"k_local<64", "k_local_xs"), (r"k_local<128", "k_local_s"),
         (r"k_local<256", "k_local_m"), (r"k_local<512", "k_local"), (r"k_small", "k_small"),
         (r"k_narrow", "k_narrow")]


def main():
    tag = sys.argv[1]
    out = {}
    for c in (2, 3, 4, 5):
        recs = json.load(open(f"gpurun_out/{tag}_ncu_cfg{c}.json"))
        per = {}
        for r in recs:
            for pat, name in NAMES:
                if re.search(pat, r["kernel"]):
                    per.setdefault(name, []).append((r["time"], r["dram_read"] + r["dram_write"]))
                    break
        cfg = {}
        for name, v in per.items():
            v.sort(reverse=True)
            cfg[name] = (v[0][1] + v[1][1]) / 2 if name == "k_wide_scatter" and len(v) > 1 else v[0][1]
        out[f"config{c}"] = cfg
    out["_source"] = (f"ncu --set full --clock-control none of one sort per config "
                      f"(profiles/capture_cfgs.sh, profiles/{tag}_ncu_cfgC.txt): "
                      "dram__bytes_read.sum + dram__bytes_write.sum of the longest launch of each "
                      "kernel; k_wide_scatter = mean of its two longest launches (root bulk-copy "
                      "variant, level 1 register-staged), matching bench.py's per-launch average")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
