"""C-ABI: the engine library loads without a GPU, exports every symbol the
headers declare, and the ctypes mirror matches the C struct layout."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

from paper_1912_04263_b200 import _abi, solver

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(ROOT, "include", h) for h in ("qpcg_b200.h", "qpcg_b200_ops.h")]


def declared():
    names = set()
    for h in HEADERS:
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(qpcg_[a-z0-9_]+)\s*\(", src):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol():
    lib = solver.load_library()
    names = declared()
    assert len(names) >= 25
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.qpcg_version().startswith(b"qpcg-b200")


def test_struct_layout_matches_header():
    probe = r'''
#include <stddef.h>
#include <stdio.h>
#include "qpcg_b200.h"
#define P(T, f) printf(#T "." #f " %zu\n", offsetof(T, f))
int main(void) {
  printf("sizeof.settings %zu\nsizeof.info %zu\nsizeof.options %zu\nsizeof.call %zu\nsizeof.rho %zu\nsizeof.csr %zu\n",
         sizeof(qpcg_settings), sizeof(qpcg_info), sizeof(qpcg_options), sizeof(qpcg_pcg_call),
         sizeof(qpcg_rho_update), sizeof(qpcg_csr_f64));
  P(qpcg_settings, lambda_pcg); P(qpcg_settings, equil_max_passes);
  P(qpcg_info, setup_seconds); P(qpcg_info, kernel_launches); P(qpcg_info, rho_final);
  P(qpcg_options, stream); P(qpcg_options, nccl_id); P(qpcg_options, nccl_ranks);
  P(qpcg_options, transport); P(qpcg_options, rendezvous_dir);
  P(qpcg_options, on_iteration); P(qpcg_options, on_iteration_user);
  P(qpcg_pcg_call, converged);
  return 0;
}'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "p.c")
        open(c, "w").write(probe)
        exe = os.path.join(d, "p")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
        out = dict(l.split() for l in subprocess.check_output([exe]).decode().splitlines())
    assert int(out["sizeof.settings"]) == C.sizeof(_abi.Settings)
    assert int(out["sizeof.info"]) == C.sizeof(_abi.Info)
    assert int(out["sizeof.options"]) == C.sizeof(_abi.Options)
    assert int(out["sizeof.call"]) == C.sizeof(_abi.PcgCall)
    assert int(out["sizeof.rho"]) == C.sizeof(_abi.RhoUpdate)
    assert int(out["sizeof.csr"]) == C.sizeof(_abi.CsrF64)
    assert int(out["qpcg_settings.lambda_pcg"]) == _abi.Settings.lambda_pcg.offset
    assert int(out["qpcg_settings.equil_max_passes"]) == _abi.Settings.equil_max_passes.offset
    assert int(out["qpcg_info.setup_seconds"]) == _abi.Info.setup_seconds.offset
    assert int(out["qpcg_info.kernel_launches"]) == _abi.Info.kernel_launches.offset
    assert int(out["qpcg_info.rho_final"]) == _abi.Info.rho_final.offset
    assert int(out["qpcg_options.stream"]) == _abi.Options.stream.offset
    assert int(out["qpcg_options.nccl_id"]) == _abi.Options.nccl_id.offset
    assert int(out["qpcg_options.nccl_ranks"]) == _abi.Options.nccl_ranks.offset
    assert int(out["qpcg_options.transport"]) == _abi.Options.transport.offset
    assert int(out["qpcg_options.rendezvous_dir"]) == _abi.Options.rendezvous_dir.offset
    assert int(out["qpcg_options.on_iteration"]) == _abi.Options.on_iteration.offset
    assert int(out["qpcg_options.on_iteration_user"]) == _abi.Options.on_iteration_user.offset
    assert int(out["qpcg_pcg_call.converged"]) == _abi.PcgCall.converged.offset


def test_default_settings_match_reference_defaults():
    lib = solver.load_library()
    s = _abi.Settings()
    lib.qpcg_default_settings(C.byref(s))
    d = _abi.default_settings()
    for f, _ in _abi.Settings._fields_:
        assert getattr(s, f) == getattr(d, f), f


def test_settings_validation_on_host():
    lib = solver.load_library()
    msg = C.create_string_buffer(256)
    s = _abi.default_settings()
    assert lib.qpcg_validate_settings(C.byref(s), msg, 256) == 0
    for field, val, text in (("alpha", 2.0, "alpha must be in (0, 2)"),
                             ("lambda_pcg", 1.0, "lambda_pcg must be in (0, 1)"),
                             ("check_interval", 0, "iteration counts must be >= 1"),
                             ("eps_equil", 0.0, "bad equilibration parameters")):
        s = _abi.default_settings()
        setattr(s, field, val)
        assert lib.qpcg_validate_settings(C.byref(s), msg, 256) == _abi.QPCG_ERR_INVALID
        assert text in msg.value.decode()


def test_settings_json_loader():
    from paper_1912_04263_b200.problem import Settings
    s = Settings.from_json('{"lambda_pcg": 0.01, "max_admm_iter": 10}')
    assert s.lambda_pcg == 0.01 and s.max_admm_iter == 10 and s.alpha == 1.6
    with pytest.raises(RuntimeError, match="unknown key"):
        Settings.from_json('{"lambda": 0.01}')  # io.hpp:201


def test_null_and_wrong_precision_arguments_fail_cleanly():
    """Argument errors surface as return codes + messages, with no GPU needed."""
    lib = solver.load_library()
    ws = C.c_void_p()
    s = _abi.default_settings()
    rc = lib.qpcg_f64_setup(C.byref(ws), None, None, None, None, None, C.byref(s), None)
    assert rc == _abi.QPCG_ERR_INVALID and not ws.value
    assert b"null" in lib.qpcg_last_error(None)
    lib.qpcg_cleanup(None)  # no-op
    assert lib.qpcg_get_pcg_calls(None, None, 0) == 0
    assert lib.qpcg_get_rho_updates(None, None, 0) == 0
    assert lib.qpcg_get_check_iterations(None, None, 0) == 0
    lib.qpcg_f64_update_rho.argtypes = [C.c_void_p, C.c_double]
    assert lib.qpcg_f64_update_rho(None, 1.0) == _abi.QPCG_ERR_INVALID
    lib.qpcg_shard_cuts.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p]
    assert lib.qpcg_shard_cuts(None, 3, 3, 2, None) == 0
    assert lib.qpcg_validate_settings(C.byref(s), None, 0) == 0
