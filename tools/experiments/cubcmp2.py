import os, subprocess, sys, tempfile
sys.path.insert(0, "/root/repo")
import paper_2604_06664_b200 as f
t = tempfile.mkdtemp()
subprocess.run(["/root/repo/paper_2604_06664_b200/foundry", "save", "--workload", "micro", "--out", t + "/cli"], check=True)
f.save(f.preset("micro"), t + "/lib")
for root, _, files in os.walk(t + "/cli"):
    for fn in files:
        a = os.path.join(root, fn); b = a.replace("/cli/", "/lib/")
        if open(a, "rb").read() != open(b, "rb").read():
            print("DIFF", fn)
            for p in (a, b):
                out = subprocess.run(["readelf", "-S", "-W", p], capture_output=True, text=True).stdout
                print("\n".join(l for l in out.splitlines() if "]" in l)[:3000])
            sys.exit(0)
print("all identical")
