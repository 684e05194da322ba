"""Embed the reference corpus and specs into a C++ translation unit (test infra).

Writes oracle/_ref/embedded.cpp (git-ignored) so that oracle/_ref/ref_tool can
run on the GPU box, where /root/reference is absent.  Nothing here lands in
the repository's tracked tree.
"""
import os
import sys


def cxx_literal(text: str) -> str:
    # chunked raw strings: MSVC-style length limits do not apply to g++, but a
    # delimiter that cannot occur in the corpus keeps it simple.
    assert ")EMBED\"" not in text
    return 'R"EMBED(' + text + ')EMBED"'


def main() -> None:
    ref, out = sys.argv[1], sys.argv[2]
    entries = []
    for sub in ("corpus/gemm", "corpus/conv", "corpus/nonidiom", "specs"):
        d = os.path.join(ref, sub)
        for name in sorted(os.listdir(d)):
            with open(os.path.join(d, name)) as f:
                entries.append((f"{sub}/{name}", f.read()))
    with open(out, "w") as f:
        f.write("#include <map>\n#include <string>\n")
        f.write("const std::map<std::string, std::string>& embedded_files() {\n")
        f.write("  static const std::map<std::string, std::string> m = {\n")
        for key, text in entries:
            f.write(f'    {{"{key}", {cxx_literal(text)}}},\n')
        f.write("  };\n  return m;\n}\n")


if __name__ == "__main__":
    main()
