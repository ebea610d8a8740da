"""Build helper: wraps trace_body.ptx into a C++ translation unit."""
import sys

src, out = sys.argv[1], sys.argv[2]
text = open(src).read()
with open(out, "w") as f:
    f.write("// generated from %s by embed_ptx.py; do not edit\n" % src.split("/")[-1])
    f.write("namespace foundry {\nconst char* trace_body_ptx() {\n    static const char k[] =\n")
    for line in text.splitlines():
        f.write('        "%s\\n"\n' % line.replace("\\", "\\\\").replace('"', '\\"'))
    f.write("        ;\n    return k;\n}\n}  // namespace foundry\n")
