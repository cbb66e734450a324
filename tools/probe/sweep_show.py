import glob, json
for f in sorted(glob.glob("gpurun_out/sweep_*.log")):
    env = open(f.replace(".log", ".env")).read().strip()
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        st = d["pipeline"]["stage_ms_per_step"]
        print(f"{env:40s} value {d['value']:9.2f}  e2e {d['e2e']['value']:9.2f}  ms {d['ms_per_step']:8.2f}  "
              + " ".join(f"{k}={v:.2f}" for k, v in st.items()))
    except Exception as ex:
        print(env, "FAILED", open(f).read()[-300:])
