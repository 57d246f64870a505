"""SM clocks and throttle reasons sampled during a timed region (bench evidence)."""

from __future__ import annotations

import statistics
import subprocess
import threading


def cuda_pci_bus_id(device: int):
    """'DDDDDDDD:BB:DD.0' of CUDA ordinal `device` (the form NVML and nvidia-smi accept),
    or None when torch cannot see the device."""
    try:
        import torch

        p = torch.cuda.get_device_properties(device)
        return f"{p.pci_domain_id:08X}:{p.pci_bus_id:02X}:{p.pci_device_id:02X}.0"
    except Exception:
        return None


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region (NVML, else nvidia-smi)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int = 0):
        """`device` is a CUDA ordinal (after CUDA_VISIBLE_DEVICES).  NVML and nvidia-smi
        enumerate GPUs in PCI order and ignore CUDA_VISIBLE_DEVICES, so the GPU is
        addressed by its PCI bus id, never by the ordinal."""
        self.device = device
        self.bus_id = cuda_pci_bus_id(device)
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _nvml_open(self):
        """NVML handle, opened before the timed region starts (init costs ~0.1 s, longer than
        a short timed region).  None if NVML is absent: nvidia-smi is polled instead."""
        try:
            import pynvml as N

            N.nvmlInit()
            if self.bus_id is None:
                raise RuntimeError("no PCI bus id for the CUDA device")
            get = getattr(N, "nvmlDeviceGetHandleByPciBusId_v2", None) or N.nvmlDeviceGetHandleByPciBusId
            h = get(self.bus_id.encode())
            self._nvml = (N, h, N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM),
                          (N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                           N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap))
            self.source = "nvml"
        except Exception as e:  # noqa: BLE001 -- any NVML failure falls back to nvidia-smi
            self._nvml = None
            self.source = "nvidia-smi"
            self.nvml_error = f"{type(e).__name__}: {e}"

    def _sample(self):
        try:
            if self._nvml:
                N, h, mx, bits = self._nvml
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append([str(sm), str(mx), "", hex(r)] +
                                 ["Active" if r & b else "Not Active" for b in bits])
            else:
                if self.bus_id is None:
                    return
                out = subprocess.run(["nvidia-smi", f"--id={self.bus_id}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([v.strip() for v in out.split(",")])
        except Exception:
            pass

    def _run(self):
        # NVML every ~2 ms (the timed region is ~0.1 s, too short for nvidia-smi's ~50 ms/query)
        period = 0.002 if self._nvml else 0.2
        while True:
            self._sample()
            if self._stop.wait(period):
                return

    def __enter__(self):
        self._nvml_open()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=6)
        if self._nvml:
            self._sample()  # the region's last clocks, however short it was
            self._nvml[0].nvmlShutdown()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows), "source": getattr(self, "source", None),
                **({"nvml_error": self.nvml_error} if getattr(self, "nvml_error", None) else {}),
                "bus_id": self.bus_id}
