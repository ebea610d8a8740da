"""Prints the fenced code block of a Markdown file whose first line names
`tag` (e.g. "// prepare_fn_demo.cpp — ..."): INTEGRATION.md's examples are
compiled verbatim from the document (test infrastructure, oracle/Makefile)."""
import sys

text = open(sys.argv[1]).read().splitlines()
tag = sys.argv[2]
inside, block = False, []
for line in text:
    if line.startswith("```"):
        if inside:
            if block and tag in block[0]:
                print("\n".join(block))
                sys.exit(0)
            inside, block = False, []
        else:
            inside = True
        continue
    if inside:
        block.append(line)
sys.exit("no code block tagged %s" % tag)
