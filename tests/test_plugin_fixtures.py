"""The plugin boundary: user targets written against the reference's
AnnealedTarget API compile unchanged against the drop-in host headers
(csrc/host/asmc/*.hpp) and fail cleanly with capability_error when sampled (there is
no CPU sampler).  The fixtures are the reference's own, read from its test sources at
test time (test_kernel.cpp:20-30 TruncatedTarget, test_engine.cpp:286-296
SpreadTarget) -- nothing is copied into this repository."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = "/root/reference/proj/tests"
HOST = os.path.join(ROOT, "paper_2408_12057_b200", "csrc", "host")
LIB = os.path.join(ROOT, "paper_2408_12057_b200", "libasmc_b200.so")


def extract_class(path, name):
    src = open(path).read()
    i = src.index(f"class {name}")
    depth, j = 0, src.index("{", i)
    for k in range(j, len(src)):
        depth += {"{": 1, "}": -1}.get(src[k], 0)
        if depth == 0:
            return src[i:src.index(";", k) + 1]
    raise ValueError(name)


MAIN = r"""
#include <cmath>
#include <cstdio>
#include <vector>

#include "asmc/engine.hpp"
#include "asmc/errors.hpp"
#include "asmc/kernel.hpp"
#include "asmc/logsum.hpp"
#include "asmc/rng.hpp"
#include "asmc/target.hpp"

using asmc::Kernel;
using asmc::KernelKind;
using asmc::RunOptions;
using asmc::ResamplePolicy;
using asmc::Schedule;

namespace {
@FIXTURES@
}  // namespace

template <class F>
int expect_capability(F f, const char* what) {
  try {
    f();
  } catch (const asmc::capability_error& e) {
    std::printf("%s: capability_error: %s\n", what, e.what());
    return 0;
  }
  std::printf("%s: no capability_error\n", what);
  return 1;
}

int main() {
  int bad = 0;
  const TruncatedTarget tt;
  const SpreadTarget st;
  // the per-point plugin API works on the host, as in the reference
  std::vector<double> x(1);
  asmc::rng::Stream s(asmc::rng::Key{1, 2, 3, 4, 0});
  tt.sample_reference(s, x);
  bad += !(std::abs(x[0]) < 1.0 && tt.log_reference(x) == -std::log(2.0));
  st.sample_reference(s, x);
  bad += !(st.log_gamma(0.5, x) == st.log_reference(x) + 0.5 * st.potential(x));
  bad += !(tt.log_reference(std::vector<double>{3.0}) == asmc::kNegInf);
  Kernel k;
  k.kind = KernelKind::identity;
  RunOptions o;
  o.n_particles = 2;
  o.policy = ResamplePolicy::never;
  bad += expect_capability([&] { asmc::run_smc(st, k, Schedule::uniform(1), o); }, "run_smc(SpreadTarget)");
  bad += expect_capability([&] { asmc::run_sais_single(tt, k, Schedule::uniform(2), o); },
                           "run_sais_single(TruncatedTarget)");
  bad += expect_capability([&] { tt.exact_sample(0.5, s, x); }, "exact_sample");
  std::printf(bad ? "FAIL\n" : "OK\n");
  return bad;
}
"""


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference sources not present")
def test_reference_fixtures_compile_and_raise_capability_error(tmp_path):
    if not os.path.exists(LIB):
        pytest.skip("library not built")
    fx = extract_class(os.path.join(REF_TESTS, "test_kernel.cpp"), "TruncatedTarget") + "\n\n" + \
        extract_class(os.path.join(REF_TESTS, "test_engine.cpp"), "SpreadTarget")
    src = tmp_path / "fixtures.cpp"
    src.write_text(MAIN.replace("@FIXTURES@", fx))
    exe = tmp_path / "fixtures"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{HOST}", f"-I{os.path.join(ROOT, 'include')}", str(src),
                    os.path.join(HOST, "asmc.cpp"), f"-L{os.path.dirname(LIB)}", "-l:libasmc_b200.so",
                    f"-Wl,-rpath,{os.path.dirname(LIB)}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr


def test_host_stream_matches_reference_stream():
    """asmc/rng.hpp's Stream is the reference's keyed stream bit for bit (the oracle's
    reference build exposes the same words)."""
    import ctypes as C
    import oracle
    from paper_2408_12057_b200 import abi
    if not oracle.available("ref", abi.RNG_XOSHIRO):
        pytest.skip("reference not built")
    ref = oracle.load("ref", abi.RNG_XOSHIRO)
    exe_src = r"""
#include <cstdio>
#include "asmc/rng.hpp"
int main() {
  asmc::rng::Stream s(asmc::rng::Key{42, 3, 17, 5, 1});
  for (int i = 0; i < 4; ++i) std::printf("%llu\n", (unsigned long long)s.next_u64());
  asmc::rng::Stream t(asmc::rng::Key{42, 3, 17, 5, 1});
  for (int i = 0; i < 3; ++i) std::printf("%.17g\n", t.normal());
}
"""
    import tempfile
    d = tempfile.mkdtemp()
    open(os.path.join(d, "s.cpp"), "w").write(exe_src)
    subprocess.run(["g++", "-std=c++20", f"-I{HOST}", os.path.join(d, "s.cpp"), "-o", os.path.join(d, "s")],
                   check=True)
    out = subprocess.run([os.path.join(d, "s")], capture_output=True, text=True).stdout.split()
    words = ref.rng_u64((42, 3, 17, 5, 1), 4)
    assert [int(v) for v in out[:4]] == [int(v) for v in words]
    normals = ref.rng_normal((42, 3, 17, 5, 1), 3)
    assert [float(v) for v in out[4:7]] == [float(v) for v in normals]
    del C
