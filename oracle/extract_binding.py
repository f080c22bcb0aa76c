"""TEST INFRASTRUCTURE ONLY — writes the first ```cpp block of INTEGRATION.md
(the binding a reference maintainer adds, proj/src/train_b200.cpp) verbatim to
the path given, so the compiled binding is exactly the documented one."""
import sys

src, dst = sys.argv[1], sys.argv[2]
text = open(src).read()
start = text.index("```cpp\n") + len("```cpp\n")
end = text.index("```", start)
open(dst, "w").write(text[start:end])
