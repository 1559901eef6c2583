"""The C++ `stabkit::` host API (include/stabkit/*.hpp) built with g++ -std=c++20 over the C ABI."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def binary(sk):
    from paper_2507_03092_b200 import _build
    path = _build.build_host()
    assert path and os.path.exists(path)
    return path


def test_headers_keep_the_reference_api():
    """Same public names as /root/reference/proj/include/stabkit/{pauli,bitvec,error,rng}.hpp."""
    inc = os.path.join(ROOT, "include", "stabkit")
    need = {
        "pauli.hpp": ["class PauliString", "static PauliString parse(", "z_at(", "x_at(", "num_qubits()", "set_sign(", "flip_sign()",
                      "x_bit(", "z_bit(", "set_pauli(", "pauli_at(", "str()", "weight()", "is_identity()", "commutes_with(",
                      "qubitwise_commutes_with(", "same_axis(", "conj_h(", "conj_s(", "conj_sdg(", "conj_cx(", "x_words()", "z_words()",
                      "product_g_sum(", "commutation_vector(", "rowsum_plus_i("],
        "bitvec.hpp": ["words_for_bits(", "tail_mask(", "struct BitVec", "get(", "set(", "count()"],
        "error.hpp": ["Error", "ParseError", "DimensionError", "UnsupportedError", "InvariantError", "line"],
        "rng.hpp": ["splitmix64(", "struct CounterRng", "bit(", "class SplitMix64", "next()", "below(", "unit()"],
    }
    for f, names in need.items():
        txt = open(os.path.join(inc, f)).read()
        for n in names:
            assert n in txt, (f, n)


def test_cpp_host_api_cpu(binary):
    r = subprocess.run([binary, "cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_host_api_gpu(binary):
    r = subprocess.run([binary, "gpu"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_row_sharded_tableau_over_nccl(sk):
    """stabkit::NcclExchange (include/stabkit/nccl_exchange.hpp): the C++ ShardedTableau driver with its three exchanges as
    ncclAllReduce(min) / ncclBroadcast / ncclAllGather on the library stream.  This box has one GPU, so the communicator has
    one rank (NCCL refuses two ranks on a device) x 3 local shards; tests/cpp/test_nccl_exchange.cpp documents the
    one-process-per-GPU launch.  Record and rows must equal the unsharded engine; an NCCL error must surface as stabkit::Error."""
    from paper_2507_03092_b200 import _build
    path = _build.build_nccl_test()
    if path is None:
        pytest.skip("nccl.h not installed")
    env = dict(os.environ, RANK="0", WORLD_SIZE="1", NCCL_DEBUG="WARN")
    r = subprocess.run([path, "7", "3", "3"], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0 and "rank 0 ok" in r.stdout and r.stdout.count("record ok rows ok") == 2, r.stdout + r.stderr
